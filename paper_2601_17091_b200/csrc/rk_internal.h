// rk_internal.h — symbols shared between the library's translation units
// (not part of the public C ABI in include/rocket_b200.h).
#pragma once
#include "../../include/rocket_b200.h"

extern "C" {
// Set the thread-local last error (rk_last_error) and return code.
int rk_set_error(int code, const char* message);
// Free the streaming runtime's cached pinned rings (rk_release_caches).
void rk_stream_release(void);
// rk_transform for pageable host x and out: the pinned-ring pipeline of
// rocket_stream.cu with the host-side copies spread over threads.
// The device counter of executed positions that rk_transform resets and
// fills for device-pointer calls on `stream`.
int rk_stream_counter(rk_bank_t bank, void* stream, unsigned long long** counter);
int rk_stream_host(rk_bank_t bank, const void* x, int32_t dtype, int64_t n, void* out, int64_t ld_out, int64_t row0,
                   int32_t fpk, int32_t mode, int64_t* executed);
}

// NVTX ranges (SURVEY §5 tracing): visible in Nsight Systems / ncu range
// filters, near-zero cost without a tool attached (header-only nvtx3).
#include <nvtx3/nvToolsExt.h>
#include <cstdio>
struct RkRange {
  explicit RkRange(const char* name) { nvtxRangePushA(name); }
  RkRange(const char* fmt, long long a, long long b) {
    char buf[96];
    std::snprintf(buf, sizeof(buf), fmt, a, b);
    nvtxRangePushA(buf);
  }
  ~RkRange() { nvtxRangePop(); }
  RkRange(const RkRange&) = delete;
  RkRange& operator=(const RkRange&) = delete;
};
