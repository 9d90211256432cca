// rocket_stream.cu — file-to-file streaming transform (rk_transform_stream).
//
// The reference's `gridrocket transform` loads the whole dataset, transforms
// it in memory and then saves the FeatureMatrix (cli.py:138-168,
// data.py:279-302, features.py:59-67).  At the BASELINE sizes the features
// are 8-80 GB, so the host copies and the disk dominate once the transform
// takes milliseconds.  Here the rows stream through a
// ring of pinned host buffers:
//
//   reader thread   pread / memcpy rows -> pinned in-slot (dtype convert,
//                   finiteness check)
//   calling thread  H2D (h2d stream) -> rk_transform (compute stream) ->
//                   D2H (d2h stream) into a pinned out-slot
//   writer thread   pwrite the out-slot at its byte offset
//
// so disk reads, both PCIe directions, the kernels and disk writes of
// different batches overlap.  Built only on the public C ABI (rk_transform
// with device pointers on our stream).
#include "../../include/rocket_b200.h"
#include "rk_internal.h"

#include <cuda_runtime.h>
#include <sys/mman.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <cerrno>
#include <condition_variable>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

namespace {

constexpr int kSlots = 3;  // pinned host slots per direction
constexpr int kDev = 2;    // device buffers per direction

struct Ring {
  int device = 0;
  size_t in_bytes = 0, out_bytes = 0;
  void* h_in[kSlots] = {};
  void* h_out[kSlots] = {};
  void* d_in[kDev] = {};
  void* d_out[kDev] = {};
  cudaStream_t h2d = nullptr, comp = nullptr, d2h = nullptr;
  cudaEvent_t h2d_done[kSlots] = {}, d2h_done[kSlots] = {};
  cudaEvent_t in_ready[kDev] = {}, in_free[kDev] = {}, out_ready[kDev] = {}, out_free[kDev] = {};
  unsigned long long* h_exec = nullptr;  // pinned: executed positions per batch
  int64_t exec_cap = 0;
};

std::mutex g_ring_mu;
std::multimap<int, Ring*> g_free_rings;  // device -> idle rings

int cuda_fail(cudaError_t e, const char* what) {
  char buf[512];
  snprintf(buf, sizeof(buf), "%s failed: %s", what, cudaGetErrorString(e));
  return rk_set_error(RK_ERR_CUDA, buf);
}

#define ST_CUDA(call)                                \
  do {                                               \
    cudaError_t e_ = (call);                         \
    if (e_ != cudaSuccess) return cuda_fail(e_, #call); \
  } while (0)

int ring_create(int device, Ring** out) {
  Ring* r = new Ring();
  r->device = device;
  ST_CUDA(cudaStreamCreateWithFlags(&r->h2d, cudaStreamNonBlocking));
  ST_CUDA(cudaStreamCreateWithFlags(&r->comp, cudaStreamNonBlocking));
  ST_CUDA(cudaStreamCreateWithFlags(&r->d2h, cudaStreamNonBlocking));
  for (int i = 0; i < kSlots; ++i) {
    ST_CUDA(cudaEventCreateWithFlags(&r->h2d_done[i], cudaEventDisableTiming));
    ST_CUDA(cudaEventCreateWithFlags(&r->d2h_done[i], cudaEventDisableTiming));
  }
  for (int i = 0; i < kDev; ++i) {
    ST_CUDA(cudaEventCreateWithFlags(&r->in_ready[i], cudaEventDisableTiming));
    ST_CUDA(cudaEventCreateWithFlags(&r->in_free[i], cudaEventDisableTiming));
    ST_CUDA(cudaEventCreateWithFlags(&r->out_ready[i], cudaEventDisableTiming));
    ST_CUDA(cudaEventCreateWithFlags(&r->out_free[i], cudaEventDisableTiming));
  }
  *out = r;
  return RK_OK;
}

void ring_free_buffers(Ring* r) {
  if (r->h_exec) cudaFreeHost(r->h_exec);
  r->h_exec = nullptr;
  r->exec_cap = 0;
  for (int i = 0; i < kSlots; ++i) {
    if (r->h_in[i]) cudaFreeHost(r->h_in[i]);
    if (r->h_out[i]) cudaFreeHost(r->h_out[i]);
    r->h_in[i] = r->h_out[i] = nullptr;
  }
  for (int i = 0; i < kDev; ++i) {
    if (r->d_in[i]) cudaFree(r->d_in[i]);
    if (r->d_out[i]) cudaFree(r->d_out[i]);
    r->d_in[i] = r->d_out[i] = nullptr;
  }
  r->in_bytes = r->out_bytes = 0;
}

void ring_destroy(Ring* r) {
  ring_free_buffers(r);
  for (int i = 0; i < kSlots; ++i) {
    cudaEventDestroy(r->h2d_done[i]);
    cudaEventDestroy(r->d2h_done[i]);
  }
  for (int i = 0; i < kDev; ++i) {
    cudaEventDestroy(r->in_ready[i]);
    cudaEventDestroy(r->in_free[i]);
    cudaEventDestroy(r->out_ready[i]);
    cudaEventDestroy(r->out_free[i]);
  }
  cudaStreamDestroy(r->h2d);
  cudaStreamDestroy(r->comp);
  cudaStreamDestroy(r->d2h);
  delete r;
}

// Grow (never shrink) the ring's buffers; cached across calls, released by
// rk_release_caches.
int ring_reserve(Ring* r, size_t in_bytes, size_t out_bytes) {
  if (in_bytes > r->in_bytes) {
    for (int i = 0; i < kSlots; ++i) {
      if (r->h_in[i]) cudaFreeHost(r->h_in[i]);
      r->h_in[i] = nullptr;
      ST_CUDA(cudaHostAlloc(&r->h_in[i], in_bytes, cudaHostAllocDefault));
    }
    for (int i = 0; i < kDev; ++i) {
      if (r->d_in[i]) cudaFree(r->d_in[i]);
      r->d_in[i] = nullptr;
      ST_CUDA(cudaMalloc(&r->d_in[i], in_bytes));
    }
    r->in_bytes = in_bytes;
  }
  if (out_bytes > r->out_bytes) {
    for (int i = 0; i < kSlots; ++i) {
      if (r->h_out[i]) cudaFreeHost(r->h_out[i]);
      r->h_out[i] = nullptr;
      ST_CUDA(cudaHostAlloc(&r->h_out[i], out_bytes, cudaHostAllocDefault));
    }
    for (int i = 0; i < kDev; ++i) {
      if (r->d_out[i]) cudaFree(r->d_out[i]);
      r->d_out[i] = nullptr;
      ST_CUDA(cudaMalloc(&r->d_out[i], out_bytes));
    }
    r->out_bytes = out_bytes;
  }
  return RK_OK;
}

// Shared progress of one streaming call.  Counters only grow; every wait
// also wakes on an error.
struct Progress {
  std::mutex mu;
  std::condition_variable cv;
  int64_t read = 0;      // batches in pinned in-slots
  int64_t h2d_enq = 0;   // batches whose H2D is enqueued (h2d_done recorded)
  int64_t d2h_enq = 0;   // batches whose D2H is enqueued (d2h_done recorded)
  int64_t written = 0;   // batches written to out_fd
  int code = RK_OK;
  std::string message;

  void set(int64_t Progress::*field, int64_t v) {
    {
      std::lock_guard<std::mutex> lk(mu);
      this->*field = v;
    }
    cv.notify_all();
  }
  // wait until this->*field > k; false on an error
  bool wait_past(int64_t Progress::*field, int64_t k) {
    std::unique_lock<std::mutex> lk(mu);
    cv.wait(lk, [&] { return code != RK_OK || this->*field > k; });
    return code == RK_OK;
  }
  void error(int c, const std::string& m) {
    {
      std::lock_guard<std::mutex> lk(mu);
      if (code == RK_OK) {
        code = c;
        message = m;
      }
    }
    cv.notify_all();
  }
};

bool read_full(int fd, void* dst, size_t bytes, int64_t offset, std::string* why) {
  char* p = static_cast<char*>(dst);
  while (bytes > 0) {
    const ssize_t got = pread(fd, p, bytes, (off_t)offset);
    if (got < 0) {
      if (errno == EINTR) continue;
      *why = std::string("read failed: ") + strerror(errno);
      return false;
    }
    if (got == 0) {
      *why = "truncated array data";
      return false;
    }
    p += got;
    bytes -= (size_t)got;
    offset += got;
  }
  return true;
}

bool write_full(int fd, const void* src, size_t bytes, int64_t offset, std::string* why) {
  const char* p = static_cast<const char*>(src);
  while (bytes > 0) {
    const ssize_t put = pwrite(fd, p, bytes, (off_t)offset);
    if (put < 0) {
      if (errno == EINTR) continue;
      *why = std::string("write failed: ") + strerror(errno);
      return false;
    }
    p += put;
    bytes -= (size_t)put;
    offset += put;
  }
  return true;
}

// Index of the first non-finite element (exponent all ones), or -1.
template <class Bits, Bits kExp>
int64_t first_nonfinite(const void* data, int64_t count) {
  const Bits* b = static_cast<const Bits*>(data);
  for (int64_t base = 0; base < count; base += 4096) {
    const int64_t end = std::min<int64_t>(count, base + 4096);
    bool any = false;
    for (int64_t i = base; i < end; ++i) any |= (b[i] & kExp) == kExp;
    if (any)
      for (int64_t i = base; i < end; ++i)
        if ((b[i] & kExp) == kExp) return i;
  }
  return -1;
}

}  // namespace

extern "C" void rk_stream_release(void) {
  std::lock_guard<std::mutex> lk(g_ring_mu);
  for (auto& kv : g_free_rings) {
    cudaSetDevice(kv.first);
    ring_destroy(kv.second);
  }
  g_free_rings.clear();
}

namespace {

// Copy `rows` rows of `row_bytes` from src (stride src_ld) to dst (stride
// dst_ld) with up to `threads` threads: the destination is usually fresh
// pageable memory, and its first-touch page faults are what bounds the copy,
// so they are taken in parallel.
void copy_rows(char* dst, int64_t dst_ld, const char* src, int64_t src_ld, int64_t row_bytes, int64_t rows,
               int threads) {
  const int64_t total = rows * row_bytes;
  auto part = [&](int64_t r0, int64_t r1) {
    if (dst_ld == row_bytes && src_ld == row_bytes) {
      std::memcpy(dst + r0 * row_bytes, src + r0 * row_bytes, (size_t)((r1 - r0) * row_bytes));
    } else {
      for (int64_t r = r0; r < r1; ++r) std::memcpy(dst + r * dst_ld, src + r * src_ld, (size_t)row_bytes);
    }
  };
  const int t = (int)std::max<int64_t>(1, std::min<int64_t>(threads, total / (4 << 20)));
  if (t <= 1 || rows < t) {
    part(0, rows);
    return;
  }
  std::vector<std::thread> pool;
  for (int i = 0; i < t; ++i) pool.emplace_back(part, rows * i / t, rows * (i + 1) / t);
  for (auto& th : pool) th.join();
}

// Where the rows come from and where the features go.
struct StreamIO {
  int in_fd = -1;             // source file (or -1: memory)
  int64_t in_offset = 0;
  const char* x = nullptr;    // source rows in memory (in_fd < 0)
  int in_dtype = RK_DTYPE_F32;
  bool check_finite = true;   // the reference's _check_shapes scan
  int out_fd = -1;            // sink file (or -1: memory)
  int64_t out_offset = 0;
  char* out = nullptr;        // sink rows in memory (out_fd < 0)
  int64_t out_ld_bytes = 0;   // sink row stride (memory)
  int copy_threads = 1;
};

int run_stream(rk_bank_t bank, const StreamIO& io, int64_t n, int32_t dtype, int32_t fpk, int32_t mode,
               int64_t batch_rows, int64_t* executed) {
  RkRange range("rk stream n=%lld mode=%lld", (long long)n, (long long)mode);
  rk_bank_info_t info;
  int rc = rk_bank_info(bank, &info);
  if (rc) return rc;
  if (n == 0) return RK_OK;
  const int64_t row_vals = (int64_t)info.n_channels * info.l_series;
  const int in_esz = io.in_dtype == RK_DTYPE_F64 ? 8 : 4;
  const int esz = dtype == RK_DTYPE_F64 ? 8 : 4;
  const int64_t in_row = row_vals * in_esz;   // bytes per row in the source
  const int64_t dev_row = row_vals * esz;     // bytes per row on the device
  const int64_t out_cols = info.n_kernels * fpk;
  const int64_t out_row = out_cols * esz;
  int64_t batch = batch_rows;
  if (batch <= 0) {
    // ~256 MB of features per batch (RK_STREAM_BATCH_MB), but never so few
    // series that the transform kernels run below a full wave of CTAs
    static const int64_t mb = getenv("RK_STREAM_BATCH_MB") ? std::max(1, atoi(getenv("RK_STREAM_BATCH_MB"))) : 256;
    batch = std::max<int64_t>(4096, (mb << 20) / std::max<int64_t>(1, out_row));
    batch = std::min<int64_t>(batch, 65535);
    // long series: bound the pinned input slots too
    batch = std::min<int64_t>(batch, std::max<int64_t>(64, ((int64_t)512 << 20) / std::max<int64_t>(1, dev_row)));
    // a few thousand rows: up to three batches of >= 1,000 rows so copies
    // overlap the kernels (as rk_transform's pinned pipeline)
    if (n < batch) {
      const int64_t k = std::max<int64_t>(1, std::min<int64_t>(3, n / 1000));
      batch = (n + k - 1) / k;
    }
  }
  batch = std::min(batch, n);
  const int64_t nb = (n + batch - 1) / batch;

  if (cudaSetDevice(info.device) != cudaSuccess) return rk_set_error(RK_ERR_CUDA, "cudaSetDevice failed");
  Ring* ring = nullptr;
  {
    std::lock_guard<std::mutex> lk(g_ring_mu);
    auto it = g_free_rings.find(info.device);
    if (it != g_free_rings.end()) {
      ring = it->second;
      g_free_rings.erase(it);
    }
  }
  if (!ring) {
    rc = ring_create(info.device, &ring);
    if (rc) return rc;
  }
  struct Return {
    Ring* r;
    ~Return() {
      std::lock_guard<std::mutex> lk(g_ring_mu);
      g_free_rings.emplace(r->device, r);
    }
  } give_back{ring};
  rc = ring_reserve(ring, (size_t)(batch * dev_row), (size_t)(batch * out_row));
  if (rc) return rc;
  if (ring->exec_cap < nb) {
    if (ring->h_exec) cudaFreeHost(ring->h_exec);
    ring->h_exec = nullptr;
    ST_CUDA(cudaHostAlloc(&ring->h_exec, sizeof(unsigned long long) * nb, cudaHostAllocDefault));
    ring->exec_cap = nb;
  }
  // the kernels count executed positions on the device, per batch
  unsigned long long* d_exec = nullptr;
  rc = rk_stream_counter(bank, (void*)ring->comp, &d_exec);
  if (rc) return rc;

  Progress pg;
  auto rows_of = [&](int64_t k) { return std::min(batch, n - k * batch); };

  std::thread reader([&] {
    cudaSetDevice(info.device);
    std::vector<char> staging;  // source-dtype rows when converting
    for (int64_t k = 0; k < nb; ++k) {
      const int s = (int)(k % kSlots);
      if (k >= kSlots) {
        if (!pg.wait_past(&Progress::h2d_enq, k - kSlots)) return;
        if (cudaEventSynchronize(ring->h2d_done[s]) != cudaSuccess) {
          pg.error(RK_ERR_CUDA, "cudaEventSynchronize(h2d) failed");
          return;
        }
      }
      const int64_t rows = rows_of(k), r0 = k * batch;
      const size_t src_bytes = (size_t)(rows * in_row);
      void* dst = ring->h_in[s];
      void* src_buf = in_esz == esz ? dst : nullptr;
      if (!src_buf) {
        staging.resize(src_bytes);
        src_buf = staging.data();
      }
      std::string why;
      if (io.in_fd >= 0) {
        if (!read_full(io.in_fd, src_buf, src_bytes, io.in_offset + r0 * in_row, &why)) {
          pg.error(RK_ERR_INVALID, why);
          return;
        }
      } else {
        std::memcpy(src_buf, io.x + r0 * in_row, src_bytes);
      }
      const int64_t count = rows * row_vals;
      if (io.check_finite) {
        const int64_t bad = in_esz == 8 ? first_nonfinite<uint64_t, 0x7ff0000000000000ull>(src_buf, count)
                                        : first_nonfinite<uint32_t, 0x7f800000u>(src_buf, count);
        if (bad >= 0) {
          char buf[160];
          snprintf(buf, sizeof(buf), "input contains non-finite values (series %lld)",
                   (long long)(r0 + bad / row_vals));
          pg.error(RK_ERR_INVALID, buf);
          return;
        }
      }
      if (in_esz != esz) {
        if (in_esz == 8) {
          const double* a = reinterpret_cast<const double*>(src_buf);
          float* b = static_cast<float*>(dst);
          for (int64_t i = 0; i < count; ++i) b[i] = (float)a[i];
        } else {
          const float* a = reinterpret_cast<const float*>(src_buf);
          double* b = static_cast<double*>(dst);
          for (int64_t i = 0; i < count; ++i) b[i] = (double)a[i];
        }
      }
      pg.set(&Progress::read, k + 1);
    }
  });

  std::thread writer([&] {
    cudaSetDevice(info.device);
    for (int64_t k = 0; k < nb; ++k) {
      const int s = (int)(k % kSlots);
      if (!pg.wait_past(&Progress::d2h_enq, k)) return;
      if (cudaEventSynchronize(ring->d2h_done[s]) != cudaSuccess) {
        pg.error(RK_ERR_CUDA, "cudaEventSynchronize(d2h) failed");
        return;
      }
      const int64_t rows = rows_of(k);
      if (io.out_fd >= 0) {
        std::string why;
        if (!write_full(io.out_fd, ring->h_out[s], (size_t)(rows * out_row), io.out_offset + k * batch * out_row,
                        &why)) {
          pg.error(RK_ERR_INVALID, why);
          return;
        }
      } else {
        copy_rows(io.out + k * batch * io.out_ld_bytes, io.out_ld_bytes, static_cast<const char*>(ring->h_out[s]),
                  out_row, out_row, rows, io.copy_threads);
      }
      pg.set(&Progress::written, k + 1);
    }
  });

  // calling thread: the GPU side
  auto gpu = [&]() -> int {
    for (int64_t k = 0; k < nb; ++k) {
      const int s = (int)(k % kSlots), db = (int)(k % kDev);
      const int64_t rows = rows_of(k);
      if (!pg.wait_past(&Progress::read, k)) return RK_OK;
      if (k >= kDev) ST_CUDA(cudaStreamWaitEvent(ring->h2d, ring->in_free[db], 0));
      ST_CUDA(cudaMemcpyAsync(ring->d_in[db], ring->h_in[s], (size_t)(rows * dev_row), cudaMemcpyHostToDevice,
                              ring->h2d));
      ST_CUDA(cudaEventRecord(ring->h2d_done[s], ring->h2d));
      ST_CUDA(cudaEventRecord(ring->in_ready[db], ring->h2d));
      pg.set(&Progress::h2d_enq, k + 1);
      ST_CUDA(cudaStreamWaitEvent(ring->comp, ring->in_ready[db], 0));
      if (k >= kDev) ST_CUDA(cudaStreamWaitEvent(ring->comp, ring->out_free[db], 0));
      const int trc = rk_transform(bank, ring->d_in[db], dtype, rows, ring->d_out[db], out_cols, 0, fpk, mode,
                                   (void*)ring->comp, nullptr);
      if (trc) return trc;
      ST_CUDA(cudaMemcpyAsync(ring->h_exec + k, d_exec, sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                              ring->comp));
      ST_CUDA(cudaEventRecord(ring->in_free[db], ring->comp));
      ST_CUDA(cudaEventRecord(ring->out_ready[db], ring->comp));
      if (k >= kSlots && !pg.wait_past(&Progress::written, k - kSlots)) return RK_OK;
      ST_CUDA(cudaStreamWaitEvent(ring->d2h, ring->out_ready[db], 0));
      ST_CUDA(cudaMemcpyAsync(ring->h_out[s], ring->d_out[db], (size_t)(rows * out_row), cudaMemcpyDeviceToHost,
                              ring->d2h));
      ST_CUDA(cudaEventRecord(ring->out_free[db], ring->d2h));
      ST_CUDA(cudaEventRecord(ring->d2h_done[s], ring->d2h));
      pg.set(&Progress::d2h_enq, k + 1);
    }
    return RK_OK;
  };
  const int grc = gpu();
  if (grc != RK_OK) pg.error(grc, rk_last_error());
  reader.join();
  writer.join();
  // drain whatever is still queued before the buffers are reused
  cudaStreamSynchronize(ring->h2d);
  cudaStreamSynchronize(ring->comp);
  cudaStreamSynchronize(ring->d2h);
  if (pg.code != RK_OK) return rk_set_error(pg.code, pg.message.c_str());
  if (executed) {
    int64_t tot = 0;
    for (int64_t k = 0; k < nb; ++k) tot += (int64_t)ring->h_exec[k];
    *executed = tot;
  }
  return RK_OK;
}

int validate_common(int32_t in_dtype, int32_t dtype, int32_t fpk, int32_t mode, int64_t n) {
  if (n < 0) return rk_set_error(RK_ERR_INVALID, "n_series must be non-negative");
  if ((in_dtype != RK_DTYPE_F32 && in_dtype != RK_DTYPE_F64) || (dtype != RK_DTYPE_F32 && dtype != RK_DTYPE_F64))
    return rk_set_error(RK_ERR_INVALID, "unknown dtype");
  if (fpk != 2 && fpk != 3) return rk_set_error(RK_ERR_INVALID, "features_per_kernel must be 2 or 3");
  if (mode != RK_MODE_EXACT && mode != RK_MODE_FAST) return rk_set_error(RK_ERR_INVALID, "unknown mode");
  return RK_OK;
}

}  // namespace

extern "C" int rk_transform_stream(rk_bank_t bank, int32_t in_fd, int64_t in_offset, const void* x,
                                   int32_t in_dtype, int64_t n, int32_t out_fd, int64_t out_offset,
                                   int32_t dtype, int32_t fpk, int32_t mode, int64_t batch_rows,
                                   int64_t* executed) {
  if (executed) *executed = 0;
  rk_bank_info_t info;
  int rc = rk_bank_info(bank, &info);
  if (rc) return rc;
  rc = validate_common(in_dtype, dtype, fpk, mode, n);
  if (rc) return rc;
  if (in_fd < 0 && !x && n > 0) return rk_set_error(RK_ERR_INVALID, "no input: in_fd < 0 and x is NULL");
  if (out_fd < 0) return rk_set_error(RK_ERR_INVALID, "out_fd must be an open file descriptor");
  if (in_offset < 0 || out_offset < 0) return rk_set_error(RK_ERR_INVALID, "negative file offset");
  StreamIO io;
  io.in_fd = in_fd;
  io.in_offset = in_offset;
  io.x = static_cast<const char*>(x);
  io.in_dtype = in_dtype;
  io.check_finite = true;
  io.out_fd = out_fd;
  io.out_offset = out_offset;
  return run_stream(bank, io, n, dtype, fpk, mode, batch_rows, executed);
}

// rk_transform's path for pageable host buffers (rk_internal.h).
extern "C" int rk_stream_host(rk_bank_t bank, const void* x, int32_t dtype, int64_t n, void* out, int64_t ld_out,
                              int64_t row0, int32_t fpk, int32_t mode, int64_t* executed) {
  if (executed) *executed = 0;
  int rc = validate_common(dtype, dtype, fpk, mode, n);
  if (rc) return rc;
  const int esz = dtype == RK_DTYPE_F64 ? 8 : 4;
  StreamIO io;
  io.x = static_cast<const char*>(x);
  io.in_dtype = dtype;
  io.check_finite = false;  // the caller validated (engine._check_shapes)
  io.out = static_cast<char*>(out) + row0 * ld_out * esz;
  io.out_ld_bytes = ld_out * esz;
  // A fresh output array (numpy's np.empty: untouched pages) is first
  // touched by the copy threads; ask for transparent huge pages so 8 GB of
  // features fault in 2 MB at a time instead of 4 KB (THP "madvise" mode;
  // a no-op for pages already present or where THP is off).
  {
    const uintptr_t huge = (uintptr_t)2 << 20;
    const uintptr_t beg = ((uintptr_t)io.out + huge - 1) & ~(huge - 1);
    const uintptr_t end = ((uintptr_t)io.out + (uintptr_t)(n * ld_out * esz)) & ~(huge - 1);
    if (end > beg) madvise((void*)beg, end - beg, MADV_HUGEPAGE);
  }
  const unsigned hw = std::thread::hardware_concurrency();
  io.copy_threads = (int)std::max(1u, std::min(16u, hw ? hw : 4u));
  if (getenv("RK_COPY_THREADS")) io.copy_threads = std::max(1, atoi(getenv("RK_COPY_THREADS")));
  return run_stream(bank, io, n, dtype, fpk, mode, 0, executed);
}
