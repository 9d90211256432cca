// rocket_b200.cu — host runtime and C ABI of the B200 ROCKET transform.
//
//  * rk_bank_create builds the dilation-grouped device bank from the
//    columnar KernelBank arrays (reference kernels.py:51-99);
//  * rk_transform_f32 runs the transform over host or device series,
//    pipelining H2D / kernel / D2H in row batches for host buffers;
//  * rk_run_batch_f32 mirrors the reference's numba entry point
//    engine._run_batch (engine.py:148-190, called at engine.py:280-295).
#include "../../include/rocket_b200.h"
#include "transform_kernel.cuh"
#include "kernel_tables.h"
#include "rk_internal.h"

#include <cuda_runtime.h>

#include <algorithm>
#include <array>
#include <atomic>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <tuple>
#include <vector>

namespace {

thread_local std::string g_last_error;

int fail(int code, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return code;
}

#define RK_CUDA(call)                                                                  \
  do {                                                                                 \
    cudaError_t e_ = (call);                                                           \
    if (e_ != cudaSuccess)                                                             \
      return fail(RK_ERR_CUDA, "%s failed: %s (%s:%d)", #call, cudaGetErrorString(e_), \
                  __FILE__, __LINE__);                                                 \
  } while (0)

// per-call device scratch: the executed counter + one item counter per class
constexpr int kMaxLaunches = 4096;
constexpr size_t kScratchBytes = sizeof(unsigned long long) + sizeof(int) * kMaxLaunches;

constexpr int kLenIdx[12] = {-1, -1, -1, -1, -1, -1, -1, 0, -1, 1, -1, 2};

struct HostChunk {
  rk::DevChunk dev;
  int64_t cost;       // instruction-slot estimate for one series
  bool tail = false;  // tail mode (the wide kernel's WChunk flag)
  int amap = -1;      // run-major lane map: log2 g (transform_kernel.cuh run_positions), -1: residue-major
};

// Shared-memory wavefronts of a chunk's complete-run steps under either lane
// map of run_positions (amap < 0: residue-major, else run-major with g =
// 2^amap), summed over up to 24 steps spread over the chunk: the largest
// number of a step's LANES run starts that share a bank (every window load
// of the step replays that many times).
int64_t lanemap_wavefronts(int d, int n, int R, int lanes, int amap) {
  const int64_t RD = (int64_t)R * d, A = n / RD, full = A * d, nfull = full / lanes;
  if (nfull == 0) return 0;
  const int64_t samples = std::min<int64_t>(nfull, 24);
  int64_t tot = 0;
  for (int64_t k = 0; k < samples; ++k) {
    const int64_t base = (nfull * k / samples) * lanes;
    int cover[32] = {};
    int mx = 0;
    for (int l = 0; l < lanes; ++l) {
      const int64_t i = base + l;
      int64_t v;
      if (amap < 0) {
        v = (i / d) * RD + i % d;
      } else {
        const int64_t g = 1LL << amap, j = i >> amap;
        v = (j % A) * RD + (j / A) * g + (i & (g - 1));
      }
      mx = std::max(mx, ++cover[v % 32]);
    }
    tot += mx;
  }
  return tot;
}

// Instruction-slot estimate of one chunk for one series at a given R
// (positions per lane, stride = dilation), following the kernel's lane map
// (run_positions): full 32-lane steps of R positions, then 1-position
// masked steps for the leftover positions.
// lanes = 16: half-warp chunks, whose steps serve two series (the caller
// halves the step part).
int64_t chunk_cost(int len, int d, int n, int nc, int P, int R, bool dyn = false, int lanes = 32, bool tail = false) {
  const int64_t G = 2 * P;
  const int64_t RD = (int64_t)R * d;
  const int64_t A = n / RD;
  const int64_t rem = n - A * RD;
  const int64_t full_starts = A * d;
  // tail mode: the R map covers the complete runs only and the remaining
  // rem positions run as an R = 1 map (no partial runs)
  const int64_t starts = tail ? full_starts : full_starts + std::min<int64_t>(d, rem);
  const int64_t nfull = full_starts / lanes;
  const int64_t masked_steps = (starts - nfull * lanes + lanes - 1) / lanes;
  auto step = [&](int64_t r, int64_t extra) {
    return r * len * nc * P              // FFMA2
           + r * G * 2                   // count (FSETP + IADD)
           + (r * G + 1) / 2             // max (FMNMX3 pairs)
           + 2 * (r + len - 1) * nc      // window loads + addresses
           + (dyn ? (P * len + 8) * nc : 0)  // run-time slots: weight reloads, slot loop
           + extra;
  };
  // a masked step adds a compare and a select per last-tap load (the
  // NaN-slot masking, transform_kernel.cuh load_window_masked)
  static const int mpct = getenv("RK_MASK_COST_PCT") ? atoi(getenv("RK_MASK_COST_PCT")) : 100;
  static const int chunk_extra = getenv("RK_CHUNK_COST") ? atoi(getenv("RK_CHUNK_COST")) : 60;
  int64_t c = nfull * step(R, 8) + masked_steps * (step(R, 18) + 4 * R * nc) * mpct / 100 + 40 * G + chunk_extra;
  if (tail && rem > 0) {
    const int64_t tf = rem / lanes, tm = (rem - tf * lanes + lanes - 1) / lanes;
    c += tf * step(1, 8) + tm * (step(1, 18) + 4 * nc) * mpct / 100;
  }
  return c;
}

// Cost of a position-paired single-kernel chunk (kinds 6 / 7): two runs of R
// positions per lane (64 run starts per step), R FFMA2 pairs per tap and
// slot, two window loads per pair slot.
int64_t chunk_cost_sp(int len, int d, int n, int nc, int R, bool tail = false) {
  auto steps = [&](int64_t nn, int64_t r, bool tl, int64_t& nfull, int64_t& masked) {
    const int64_t RD = r * d, A = nn / RD, rem = nn - A * RD, full_starts = A * d;
    const int64_t starts = tl ? full_starts : full_starts + std::min<int64_t>(d, rem);
    nfull = full_starts / 64;
    masked = (starts - nfull * 64 + 63) / 64;
    return rem;
  };
  auto step = [&](int64_t r, int64_t extra) {
    return r * len * nc              // FFMA2
           + 2 * r * 2               // count (2r outputs)
           + r                       // max (FMNMX3 pairs)
           + 4 * (r + len - 1) * nc  // two window loads + addresses per pair slot
           + extra;
  };
  static const int chunk_extra = getenv("RK_CHUNK_COST") ? atoi(getenv("RK_CHUNK_COST")) : 60;
  int64_t nf = 0, nm = 0;
  const int64_t rem = steps(n, R, tail && R > 1, nf, nm);
  int64_t c = nf * step(R, 8) + nm * (step(R, 18) + 8LL * R * nc) + 40 * 2 + chunk_extra;
  if (tail && R > 1 && rem > 0) {
    int64_t f1 = 0, m1 = 0;
    steps(rem, 1, false, f1, m1);
    c += f1 * step(1, 8) + m1 * (step(1, 18) + 8LL * nc);
  }
  return c;
}

}  // namespace

struct rk_bank_s {
  int device = 0;
  int64_t K = 0;
  int C = 0, L = 0;
  int halo = 0;
  int sstride = 0;
  int smem_bytes = 0;
  int n_groups = 0;
  int64_t positions = 0;
  int64_t useful_flops = 0;
  std::vector<HostChunk> chunks;  // class-sorted
  std::vector<int64_t> cost_prefix;
  int cls_begin[rk::kNumClasses] = {};
  int cls_end[rk::kNumClasses] = {};
  // wide path: per-launch parameter blocks, built once
  struct WideLaunch {
    int cls;
    int n_chunks;
    int64_t dense_flops;  // 2 * taps * positions of one series (diagnostics)
    std::vector<rk::float4_t> blob;       // exact mode
    std::vector<rk::float4_t> blob_fast;  // fast mode: weights negated (the series is staged as is)
  };
  bool wide_path = false;  // parameter-block launches, W warps share a series
  bool gmem = false;       // series too long for shared memory: windows read from zero-haloed rows in global memory
  int wide_ctas_per_sm = 0;  // default CTAs per SM (many series)
  int wide_ctas_smem = 0;    // shared-memory limit of CTAs per SM
  std::vector<WideLaunch> wide_launches;
  rk::DevChunk* d_chunks = nullptr;
  float* d_weights = nullptr;
  int* d_chan_off = nullptr;
  // cell path (precision "double", MPV): reference-layout parameters
  rk::CellKernel* d_cell = nullptr;
  int* d_chidx = nullptr;
  float* d_cw32 = nullptr;
  float* d_cb32 = nullptr;
  double* d_cw64 = nullptr;
  double* d_cb64 = nullptr;
  std::vector<int64_t> cell_order;  // sorted position -> bank index
  int64_t cell_len_begin[3] = {}, cell_len_end[3] = {};  // sorted range per length 7/9/11
  int64_t n_weights = 0;
  int64_t device_bytes = 0;
  std::map<std::pair<int, int>, int*> d_block_start;  // (class, n_blocks) -> device boundaries
  std::mutex mu;
  std::atomic<bool> f64_ready{false};  // d_cw64 / d_cb64 filled (rk_bank_attach_f64)
  // the same bank without half-warp chunks, for transforms whose items hold
  // one series (null when the bank has no half-warp chunks)
  // the same bank limited to 1 / 2 / 4 series per pass (narrow[0]: no lane
  // groups — items of one series; narrow[1]: up to half-warp chunks —
  // items of two or three series; narrow[2]: up to quarter-warp chunks —
  // items of four to seven series); null when not narrower than this layout
  rk_bank_s* narrow[3] = {};
  // the same bank with the exact-mode lane-group margin (null when equal to
  // the fast-mode layout's or without lane-group chunks)
  rk_bank_s* exact_bank = nullptr;
  // largest series per pass of any chunk of this layout (1, 2, 4, 8)
  int max_groups = 1;

  ~rk_bank_s() {
    for (auto* t : narrow) delete t;
    delete exact_bank;
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(device);
    cudaFree(d_chunks);
    cudaFree(d_weights);
    cudaFree(d_chan_off);
    cudaFree(d_cell);
    cudaFree(d_chidx);
    cudaFree(d_cw32);
    cudaFree(d_cb32);
    cudaFree(d_cw64);
    cudaFree(d_cb64);
    for (auto& kv : d_block_start) cudaFree(kv.second);
    cudaSetDevice(prev);
  }

  // Partition class cls's chunk range into nb blocks of near-equal cost.
  int blocks_for(int cls, int nb, int** out) {
    std::lock_guard<std::mutex> lk(mu);
    auto key = std::make_pair(cls, nb);
    auto it = d_block_start.find(key);
    if (it != d_block_start.end()) {
      *out = it->second;
      return RK_OK;
    }
    const int cb = cls_begin[cls], ce = cls_end[cls];
    std::vector<int> bs(nb + 1, cb);
    const int64_t base = cost_prefix[cb], total = cost_prefix[ce] - base;
    int ci = cb;
    for (int b = 1; b < nb; ++b) {
      const int64_t target = base + total * b / nb;
      while (ci < ce && cost_prefix[ci + 1] <= target) ++ci;
      bs[b] = std::max(ci, bs[b - 1]);
    }
    bs[nb] = ce;
    int* d = nullptr;
    RK_CUDA(cudaMalloc(&d, sizeof(int) * (nb + 1)));
    RK_CUDA(cudaMemcpy(d, bs.data(), sizeof(int) * (nb + 1), cudaMemcpyHostToDevice));
    d_block_start[key] = d;
    *out = d;
    return RK_OK;
  }
};

namespace {

// Host-buffer transforms run on a pooled "worker": two streams, two events
// and double-buffered device scratch, reused across calls (per-call
// allocation made the stream-ordered pool map and unmap memory every call).
// Pipeline: h2d stream -> compute stream -> d2h stream, 3 input and 2
// output buffers; H2D of batch k+1 is enqueued before the D2H of batch k so
// a copy engine never holds the next input behind a long feature copy.
constexpr int kInBufs = 3, kOutBufs = 2;
struct Worker {
  cudaStream_t stream = nullptr, h2d_stream = nullptr, d2h_stream = nullptr;
  cudaEvent_t in_ready[kInBufs] = {}, in_free[kInBufs] = {};
  cudaEvent_t out_ready[kOutBufs] = {}, out_free[kOutBufs] = {};
  unsigned long long* d_scratch = nullptr;
  float* d_in[kInBufs] = {};
  float* d_out[kOutBufs] = {};
  size_t in_cap = 0, out_cap = 0;
};

struct DeviceState {
  int sms = 0;
  size_t smem_optin = 0;
  cudaStream_t stream = nullptr;
  std::map<const void*, int> attr_smem;
  std::mutex attr_mu;
  std::mutex pool_mu;
  std::vector<Worker*> free_workers;
  // device-pointer calls: one scratch block per stream (stream order makes
  // reuse safe)
  std::map<cudaStream_t, unsigned long long*> stream_scratch;
  // one transform's counter reset, launch chain and counter read at a time
  // per stream: concurrent callers on one stream (e.g. the library's default
  // stream) must not interleave them
  std::map<cudaStream_t, std::unique_ptr<std::mutex>> stream_mu;
  // GMEM banks: zero-haloed series rows (+ a canonical NaN) per stream
  struct Rows {
    float* p = nullptr;
    size_t floats = 0;
    int64_t layout = -1;  // (C, L, stride, halo) the halos were zeroed for
  };
  std::map<cudaStream_t, Rows> gmem_rows;
};
std::mutex g_dev_mu;
std::map<int, DeviceState*> g_devs;

int device_state(int device, DeviceState** out) {
  std::lock_guard<std::mutex> lk(g_dev_mu);
  auto it = g_devs.find(device);
  if (it == g_devs.end()) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
      cudaGetLastError();
      return fail(RK_ERR_NO_DEVICE, "no CUDA device is visible");
    }
    if (device < 0 || device >= n) return fail(RK_ERR_INVALID, "device %d out of range [0, %d)", device, n);
    RK_CUDA(cudaSetDevice(device));
    cudaDeviceProp prop;
    RK_CUDA(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10)
      return fail(RK_ERR_UNSUPPORTED, "device %d is sm_%d%d; this library is built for sm_100a (B200)", device,
                  prop.major, prop.minor);
    DeviceState* st = new DeviceState();
    st->sms = prop.multiProcessorCount;
    st->smem_optin = prop.sharedMemPerBlockOptin;
    RK_CUDA(cudaStreamCreateWithFlags(&st->stream, cudaStreamNonBlocking));
    it = g_devs.emplace(device, st).first;
  }
  *out = it->second;
  return RK_OK;
}

// Kernel tables: one instantiation per (class, mode), compiled per kernel
// length in kernels_len.cu (three translation units, built in parallel).
using rk::KernelFn;
using rk::WarpFn;
struct KernelTable {
  KernelFn fn[2 * rk::kNumClasses] = {};
  WarpFn dfn[2 * rk::kNumClasses] = {};
  WarpFn mfn[rk::kNumClasses] = {};      // fast-mode MPV wide kernels
  WarpFn gfn[2 * rk::kNumClasses] = {};  // series in global memory (GMEM)
  KernelTable() {
#define RK_FILL(L, R) rk_fill_tables_##L##_##R(fn, dfn, mfn, gfn);
#define RK_FILL_L(L) RK_FILL(L, 0) RK_FILL(L, 1) RK_FILL(L, 2) RK_FILL(L, 3) RK_FILL(L, 4) RK_FILL(L, 5) \
    RK_FILL(L, 6) RK_FILL(L, 7)
    RK_FILL_L(7)
    RK_FILL_L(9)
    RK_FILL_L(11)
#undef RK_FILL_L
#undef RK_FILL
  }
};
const KernelTable& kernel_table() {
  static KernelTable t;
  return t;
}

int stream_scratch(DeviceState* st, cudaStream_t stream, unsigned long long** out) {
  std::lock_guard<std::mutex> lk(st->pool_mu);
  auto it = st->stream_scratch.find(stream);
  if (it == st->stream_scratch.end()) {
    unsigned long long* p = nullptr;
    RK_CUDA(cudaMalloc(&p, kScratchBytes));
    it = st->stream_scratch.emplace(stream, p).first;
  }
  *out = it->second;
  return RK_OK;
}

int acquire_worker(DeviceState* st, Worker** out) {
  {
    std::lock_guard<std::mutex> lk(st->pool_mu);
    if (!st->free_workers.empty()) {
      *out = st->free_workers.back();
      st->free_workers.pop_back();
      return RK_OK;
    }
  }
  Worker* w = new Worker();
  RK_CUDA(cudaStreamCreateWithFlags(&w->stream, cudaStreamNonBlocking));
  RK_CUDA(cudaStreamCreateWithFlags(&w->h2d_stream, cudaStreamNonBlocking));
  RK_CUDA(cudaStreamCreateWithFlags(&w->d2h_stream, cudaStreamNonBlocking));
  for (int i = 0; i < kInBufs; ++i) {
    RK_CUDA(cudaEventCreateWithFlags(&w->in_ready[i], cudaEventDisableTiming));
    RK_CUDA(cudaEventCreateWithFlags(&w->in_free[i], cudaEventDisableTiming));
  }
  for (int i = 0; i < kOutBufs; ++i) {
    RK_CUDA(cudaEventCreateWithFlags(&w->out_ready[i], cudaEventDisableTiming));
    RK_CUDA(cudaEventCreateWithFlags(&w->out_free[i], cudaEventDisableTiming));
  }
  RK_CUDA(cudaMalloc(&w->d_scratch, kScratchBytes));
  *out = w;
  return RK_OK;
}

void release_worker(DeviceState* st, Worker* w) {
  std::lock_guard<std::mutex> lk(st->pool_mu);
  st->free_workers.push_back(w);
}

int set_kernel_smem(DeviceState* st, const void* fn, int bytes) {
  std::lock_guard<std::mutex> lk(st->attr_mu);
  auto it = st->attr_smem.find(fn);
  if (it == st->attr_smem.end() || it->second < bytes) {
    RK_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
    st->attr_smem[fn] = bytes;
  }
  return RK_OK;
}

bool is_device_pointer(const void* p) {
  cudaPointerAttributes attr;
  if (cudaPointerGetAttributes(&attr, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return attr.type == cudaMemoryTypeDevice || attr.type == cudaMemoryTypeManaged;
}

// Host memory the driver can DMA directly (cudaHostAlloc / registered).
bool is_pinned_host(const void* p) {
  cudaPointerAttributes attr;
  if (cudaPointerGetAttributes(&attr, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return attr.type == cudaMemoryTypeHost;
}

// The class a launch executes: exact mode (and fast MPV) run classes above
// R = kExactRMax with that R (same chunks, only positions per lane differ).
int exec_cls(int cls, int exact) {
  const int nck = cls % rk::kNumNck;
  const int ri = (cls / rk::kNumNck) % rk::kNumR;
  const int li = cls / (rk::kNumNck * rk::kNumR);
  const int r = exact && rk::r_of(ri) > rk::kExactRMax ? rk::kExactRIdx13 : ri;
  return (li * rk::kNumR + r) * rk::kNumNck + nck;
}

int c_len(int cls) { return 7 + 2 * (cls / (rk::kNumNck * rk::kNumR)); }

// Wide path: one PDL-chained launch per parameter block, all on `stream`.
int launch_wide_chain(rk_bank_t b, DeviceState* st, const float* d_x, int64_t n, float* d_out, int64_t ld_out,
                      int fpk, int mode, cudaStream_t stream, unsigned long long* d_exec, int* d_counters,
                      const float* xpad, const float* nanp) {
  const int exact = mode == RK_MODE_EXACT ? 1 : 0;
  static const bool profile = getenv("RK_PROFILE") != nullptr;
  // 32 KB parameter block, one per host thread (kept off the stack; the
  // launch copies it, so concurrent callers on other devices or streams
  // never share or wait for it)
  static thread_local rk::WParams params;
  const int smem = b->gmem ? 0 : b->smem_bytes;
  // Few series: more, narrower CTAs (down to one warp) so every SM still has
  // work; many series: wide_ctas_per_sm CTAs of 24/ctas warps.
  int ctas = b->wide_ctas_per_sm;
  if (n < 4LL * st->sms * ctas) ctas = std::min(b->wide_ctas_smem, rk::kWideMaxWarps);
  // several series per item when they fit at the same CTA count: each
  // chunk's weights and setup serve all of them
  const int spi_max = getenv("RK_SPI") ? std::max(1, atoi(getenv("RK_SPI"))) : 8;
  const int64_t min_items_env = getenv("RK_MIN_ITEMS") ? atoi(getenv("RK_MIN_ITEMS")) : 0;
  auto spi_for = [&](int c, int64_t min_items) {
    int v = 1;
    while (v < spi_max && n >= min_items * (v + 1) * st->sms * c &&
           (int64_t)c * ((v + 1) * (int64_t)smem + 1024) <= (int64_t)st->smem_optin + 1024)
      ++v;
    return v;
  };
  auto pass_width = [&](int v) {  // series per pass an item of v series fills in this layout
    int w = 1;
    while (w * 2 <= v && w * 2 <= b->max_groups) w *= 2;
    return w;
  };
  int spi = spi_for(ctas, min_items_env ? min_items_env : 2);
  // A layout with lane groups wider than the items can fill: try fewer,
  // wider CTAs (down to 2) and one item per CTA slot, keeping the CTA count
  // that fills the widest groups (FordA shape: 3 x 8 warps with 4-series
  // items -> 2 x 12 with 8-series items, eighth-warp chunks: +3.4 %).
  if (!min_items_env && b->max_groups > 1 && pass_width(spi) < b->max_groups && !getenv("RK_WIDE_CTAS")) {
    int best_c = ctas, best_v = spi;
    for (int c = ctas; c >= 2; --c) {
      const int v = spi_for(c, c == ctas ? 2 : 1);
      if (pass_width(v) > pass_width(best_v)) {
        best_c = c;
        best_v = v;
      }
    }
    ctas = best_c;
    spi = best_v;
  }
  const int warps = std::max(1, rk::kWideMaxWarps / ctas);
  // whole passes of the lane groups: no shadowed groups in the last pass of
  // an item (a 6-series item on quarter-warp chunks wasted 1/4 of a pass:
  // config 2 at 4 CTAs 240k -> 314k series/s); RK_SPI_ROUND=0 disables
  static const bool spi_round = !getenv("RK_SPI_ROUND") || atoi(getenv("RK_SPI_ROUND"));
  int pow2 = 1;  // largest power of two <= spi (series per pass an item can fill)
  while (pow2 * 2 <= spi && pow2 < 8) pow2 *= 2;
  if (spi_round && b->max_groups > 1) spi -= spi % std::min(b->max_groups, pow2);
  // one series per item: lane-group chunks cannot pair series, so run the
  // bank's full-warp twin
  if (spi < 2 && b->narrow[0])
    return launch_wide_chain(b->narrow[0], st, d_x, n, d_out, ld_out, fpk, mode, stream, d_exec, d_counters, xpad,
                             nanp);
  // exact mode: the layout priced with its own lane-group margin
  if (exact && fpk == 2 && b->exact_bank)
    return launch_wide_chain(b->exact_bank, st, d_x, n, d_out, ld_out, fpk, mode, stream, d_exec, d_counters, xpad,
                             nanp);
  // items that cannot fill the widest groups of this layout: the layout
  // priced without them
  if (pow2 < b->max_groups) {
    const int j = pow2 >= 4 ? 2 : pow2 >= 2 ? 1 : 0;
    if (b->narrow[j])
      return launch_wide_chain(b->narrow[j], st, d_x, n, d_out, ld_out, fpk, mode, stream, d_exec, d_counters, xpad,
                               nanp);
  }
  const int64_t grid = std::min<int64_t>((n + spi - 1) / spi, (int64_t)st->sms * ctas);
  RkRange range("rk launch chain spi=%lld launches=%lld", (long long)spi, (long long)b->wide_launches.size());
  if (profile)
    fprintf(stderr, "RK_PROFILE chain n=%lld spi=%d ctas=%d warps=%d launches=%zu max_groups=%d exact_twin=%d\n",
            (long long)n, spi, ctas, warps, b->wide_launches.size(), b->max_groups, b->exact_bank != nullptr);
  std::vector<cudaEvent_t> evs;
  for (size_t li = 0; li < b->wide_launches.size(); ++li) {
    const auto& wl = b->wide_launches[li];
    // fpk 3 in fast mode: MPV kernels (R capped like exact mode);
    // GMEM banks: the global-memory variants (2-pair chunks at R <= 5)
    WarpFn fn = nullptr;
    if (b->gmem) {
      int gc = exec_cls(wl.cls, exact);
      const int gnck = gc % rk::kNumNck, gri = (gc / rk::kNumNck) % rk::kNumR;
      if (gnck == 0 && gri > 2) gc += (2 - gri) * rk::kNumNck;
      fn = kernel_table().gfn[2 * gc + exact];
    } else {
      int cls = wl.cls;
      // half-warp chunks need two series per item; otherwise run their data
      // on the full-warp kernel of the same (length, R, pairs)
      // (without a twin) run lane groups the item cannot fill on the next
      // narrower kind of the same (length, R, pairs)
      while (rk::nck_groups(cls % rk::kNumNck) > std::max(1, spi)) {
        const int k = cls % rk::kNumNck;
        const int narrower = (k == 10) ? 8 : (k == 11) ? 9 : (k == 8) ? 4 : (k == 9) ? 5 : rk::nck_full(k);
        cls += narrower - k;
      }
      fn = fpk == 3 ? kernel_table().mfn[exec_cls(cls, 1)] : kernel_table().dfn[2 * exec_cls(cls, exact) + exact];
    }
    if (!fn) return fail(RK_ERR_UNSUPPORTED, "no wide kernel for class %d", wl.cls);
    int rc = set_kernel_smem(st, (const void*)fn, smem * spi);
    if (rc) return rc;
    const int nck = wl.cls % rk::kNumNck;
    const int P = rk::nck_pairs(nck), NC = std::max(1, rk::nck_slots(nck));
    const int len = c_len(wl.cls);
    rk::WHeader& h = params.h;
    h.x = d_x;
    h.out = d_out;
    h.executed = d_exec;
    h.item_counter = d_counters + li;
    h.ld_out = ld_out;
    h.n_series = n;
    h.n_chunks = wl.n_chunks;
    h.l_series = b->L;
    h.n_channels = b->C;
    h.halo = b->halo;
    h.sstride = b->sstride;
    h.fpk = fpk;
    h.vec_out = (fpk == 2 && (ld_out % 2) == 0 && ((uintptr_t)d_out % 8) == 0) ? 1 : 0;
    h.vec_in = ((b->L % 4) == 0 && ((uintptr_t)d_x % 16) == 0 && (b->sstride % 4) == 0 && (b->halo % 4) == 0) ? 1 : 0;
    h.one = 1.0f;
    h.wbytes = NC * P * len * 8;
    h.spi = spi;
    h.xpad = xpad;
    h.nanp = nanp;
    std::memcpy(params.blob, exact ? wl.blob.data() : wl.blob_fast.data(), sizeof(params.blob));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3(32 * warps);
    cfg.dynamicSmemBytes = smem * spi;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = li == 0 ? 0 : 1;  // the first launch follows the counter memset normally
    if (profile) {
      cudaEvent_t e;
      cudaEventCreate(&e);
      cudaEventRecord(e, stream);
      evs.push_back(e);
      cfg.numAttrs = 0;
    }
    void* args[] = {&params};
    RK_CUDA(cudaLaunchKernelExC(&cfg, (const void*)fn, args));
  }
  if (profile) {
    cudaEvent_t e;
    cudaEventCreate(&e);
    cudaEventRecord(e, stream);
    evs.push_back(e);
    cudaEventSynchronize(e);
    for (size_t i = 0; i + 1 < evs.size(); ++i) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, evs[i], evs[i + 1]);
      const auto& wl = b->wide_launches[i];
      fprintf(stderr, "RK_PROFILE wide len=%d R=%d nck=%d exact=%d chunks=%d grid=%lld ms=%.3f dense_tflops=%.2f\n",
              c_len(wl.cls), rk::r_of((wl.cls / rk::kNumNck) % rk::kNumR), wl.cls % rk::kNumNck, exact,
              wl.n_chunks, (long long)grid, ms, wl.dense_flops * (double)n / (ms * 1e-3) / 1e12);
    }
    for (auto e : evs) cudaEventDestroy(e);
  }
  return RK_OK;
}

int padded_rows(rk_bank_t b, DeviceState* st, cudaStream_t stream, int esz, const void* d_x, int64_t rows,
                void** out);

// Wide path entry: GMEM banks copy each batch of series into zero-haloed
// rows in a per-stream scratch (halos zeroed once, interiors by a 2-D
// copy) and run the chain per batch; other banks run the chain directly.
int launch_wide(rk_bank_t b, DeviceState* st, const float* d_x, int64_t n, float* d_out, int64_t ld_out, int fpk,
                int mode, cudaStream_t stream, unsigned long long* d_exec, int* d_counters) {
  if (!b->gmem) return launch_wide_chain(b, st, d_x, n, d_out, ld_out, fpk, mode, stream, d_exec, d_counters,
                                         nullptr, nullptr);
  const int64_t row_floats = (int64_t)b->C * b->sstride;
  const int64_t budget = ((int64_t)1 << 30) / 4;  // 1 GB of padded rows per batch
  const int64_t batch = std::max<int64_t>(1, std::min<int64_t>(n, budget / row_floats));
  for (int64_t s0 = 0; s0 < n; s0 += batch) {
    const int64_t cnt = std::min(batch, n - s0);
    void* rows = nullptr;
    int rc = padded_rows(b, st, stream, 4, d_x + s0 * b->C * b->L, cnt, &rows);
    if (rc) return rc;
    const float* xpad = static_cast<const float*>(rows);
    const float* nanp = nullptr;
    {
      std::lock_guard<std::mutex> lk(st->pool_mu);
      const auto& r = st->gmem_rows[stream];
      nanp = r.p + r.floats - 1;
    }
    if (s0 > 0) RK_CUDA(cudaMemsetAsync(d_counters, 0, sizeof(int) * kMaxLaunches, stream));
    rc = launch_wide_chain(b, st, d_x, cnt, d_out + s0 * ld_out, ld_out, fpk, mode, stream, d_exec, d_counters,
                           xpad, nanp);
    if (rc) return rc;
  }
  return RK_OK;
}

// Cell path: float64 (precision "double") and exact MPV (fpk = 3): the
// reference loop order on the CUDA cores.  The staged cell kernel (one
// series in shared memory, one launch per kernel length) when a series fits;
// otherwise the same kernel reading zero-haloed rows from global memory
// (RK_NO_CELLROW: the unstaged thread-per-cell kernel).
#ifndef RK_CELL_B
#define RK_CELL_B 4  // positions per block (independent accumulation chains)
#endif
template <typename T, bool MPV, int LEN, bool GMEM>
int launch_cellrow(DeviceState* st, const rk::CellArgs& a, size_t smem, cudaStream_t stream) {
  auto fn = rk::rocket_cellrow_kernel<T, MPV, LEN, RK_CELL_B, GMEM>;
  int rc = set_kernel_smem(st, (const void*)fn, (int)smem);
  if (rc) return rc;
  int per_sm = 1;
  RK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, 256, smem));
  const int64_t grid = std::min<int64_t>(a.n_series, (int64_t)st->sms * std::max(1, per_sm));
  fn<<<(unsigned)grid, 256, smem, stream>>>(a);
  RK_CUDA(cudaGetLastError());
  return RK_OK;
}

// Position-paired cell kernel: two staged copies of the series (copy 1
// shifted by one element) so every (x[e], x[e+1]) pair is one aligned load.
template <typename T, bool MPV, int LEN>
int launch_cellpair(DeviceState* st, const rk::CellArgs& a, size_t smem, cudaStream_t stream) {
  auto fn = rk::rocket_cellpair_kernel<T, MPV, LEN>;
  int rc = set_kernel_smem(st, (const void*)fn, (int)smem);
  if (rc) return rc;
  int per_sm = 1;
  RK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, 256, smem));
  const int64_t grid = std::min<int64_t>(a.n_series, (int64_t)st->sms * std::max(1, per_sm));
  fn<<<(unsigned)grid, 256, smem, stream>>>(a);
  RK_CUDA(cudaGetLastError());
  return RK_OK;
}

// Row stride of the cell kernels' own staging: 32-float rounding plus 12,
// so the C channel rows start 12 banks apart in float32 and 24 in float64
// (lanes of one warp read different channels at once).  The wide kernel's
// pad (chosen for its lane groups, 16 at C = 3) puts float64 channel rows on
// the same banks: config 5 float64 ran 32 % slower with it (pad sweep in
// profiles/r02_cell_kernels.txt).  RK_CELL_PAD: another pad (floats,
// multiple of 2; diagnostics).
int64_t cell_sstride(rk_bank_t b) {
  static const int pad = getenv("RK_CELL_PAD") ? std::max(0, atoi(getenv("RK_CELL_PAD")) / 2 * 2) : 12;
  return (((int64_t)b->L + 2 * b->halo + 31) / 32) * 32 + pad;
}

template <typename T, bool MPV, bool GMEM>
int launch_cellrows(rk_bank_t b, DeviceState* st, rk::CellArgs a, cudaStream_t stream, int* d_counters) {
  const int64_t cs = GMEM ? b->sstride : cell_sstride(b);  // GMEM: the zero-haloed rows' stride
  const size_t smem = GMEM ? 0 : (size_t)b->C * cs * sizeof(T);
  // the paired kernel when its two copies leave room for two CTAs per SM
  const size_t psmem = 2 * smem + rk::kCellPairSlack * sizeof(T);  // two copies + dead-read slack
  const bool paired = !GMEM && !getenv("RK_NO_CELLPAIR") && 2 * (psmem + 1024) <= st->smem_optin + 1024;
  RK_CUDA(cudaMemsetAsync(d_counters, 0, sizeof(int) * 3, stream));
  a.halo = b->halo;
  a.sstride = (int)cs;
  a.one = 1.0f;
  for (int li = 0; li < 3; ++li) {
    if (b->cell_len_end[li] <= b->cell_len_begin[li]) continue;
    a.k_begin = (int)b->cell_len_begin[li];
    a.k_end = (int)b->cell_len_end[li];
    a.item_counter = d_counters + li;
    int rc;
    if (paired)
      rc = li == 0 ? launch_cellpair<T, MPV, 7>(st, a, psmem, stream)
         : li == 1 ? launch_cellpair<T, MPV, 9>(st, a, psmem, stream)
                   : launch_cellpair<T, MPV, 11>(st, a, psmem, stream);
    else
      rc = li == 0 ? launch_cellrow<T, MPV, 7, GMEM>(st, a, smem, stream)
         : li == 1 ? launch_cellrow<T, MPV, 9, GMEM>(st, a, smem, stream)
                   : launch_cellrow<T, MPV, 11, GMEM>(st, a, smem, stream);
    if (rc) return rc;
  }
  return RK_OK;
}

// Zero-haloed rows of `esz`-byte elements for `rows` series in a per-stream
// scratch: halos zeroed when the buffer grows or the layout changes, row
// interiors by one 2-D copy per call.
int padded_rows(rk_bank_t b, DeviceState* st, cudaStream_t stream, int esz, const void* d_x, int64_t rows,
                void** out) {
  const int64_t row_elems = (int64_t)b->C * b->sstride;
  const size_t need = (size_t)(rows * row_elems + 4) * esz;
  DeviceState::Rows* r = nullptr;
  {
    std::lock_guard<std::mutex> lk(st->pool_mu);
    r = &st->gmem_rows[stream];
  }
  const int64_t layout = ((((int64_t)b->C * 1000003 + b->L) * 1000003 + b->sstride) * 1000003 + b->halo) * 16 + esz;
  if (r->floats * sizeof(float) < need || r->layout != layout) {
    if (r->floats * sizeof(float) < need) {
      if (r->p) RK_CUDA(cudaFree(r->p));
      r->p = nullptr;
      RK_CUDA(cudaMalloc(&r->p, need));
      r->floats = need / sizeof(float);
    }
    RK_CUDA(cudaMemsetAsync(r->p, 0, r->floats * sizeof(float), stream));
    const float qnan = __builtin_nanf("");
    RK_CUDA(cudaMemcpyAsync(r->p + r->floats - 1, &qnan, sizeof(float), cudaMemcpyHostToDevice, stream));
    RK_CUDA(cudaStreamSynchronize(stream));
    r->layout = layout;
  }
  RK_CUDA(cudaMemcpy2DAsync(reinterpret_cast<char*>(r->p) + (size_t)b->halo * esz, (size_t)b->sstride * esz, d_x,
                            (size_t)b->L * esz, (size_t)b->L * esz, (size_t)(rows * b->C), cudaMemcpyDeviceToDevice,
                            stream));
  *out = r->p;
  return RK_OK;
}

// Cell kernels over series too long for shared memory: batches of padded
// rows in global memory (1 GB of rows per batch).
template <typename T, bool MPV>
int launch_cellrows_gmem(rk_bank_t b, DeviceState* st, rk::CellArgs a, cudaStream_t stream, int* d_counters) {
  const int64_t row_elems = (int64_t)b->C * b->sstride;
  const int64_t batch = std::max<int64_t>(1, std::min<int64_t>(a.n_series, (((int64_t)1 << 30) / sizeof(T)) /
                                                                            row_elems));
  const int64_t n = a.n_series;
  for (int64_t s0 = 0; s0 < n; s0 += batch) {
    const int64_t cnt = std::min(batch, n - s0);
    void* rows = nullptr;
    int rc = padded_rows(b, st, stream, (int)sizeof(T), static_cast<const T*>(a.x) + s0 * b->C * b->L, cnt, &rows);
    if (rc) return rc;
    rk::CellArgs ab = a;
    ab.n_series = cnt;
    ab.xpad = rows;
    ab.out = static_cast<T*>(a.out) + s0 * a.ld_out;
    rc = launch_cellrows<T, MPV, true>(b, st, ab, stream, d_counters);
    if (rc) return rc;
  }
  return RK_OK;
}

int launch_cells(rk_bank_t b, DeviceState* st, const void* d_x, int esz, int64_t n, void* d_out, int64_t ld_out,
                 int fpk, cudaStream_t stream, unsigned long long* d_exec, int* d_counters) {
  if (esz == 8 && !b->f64_ready.load(std::memory_order_acquire))
    return fail(RK_ERR_INVALID, "double precision needs rk_bank_attach_f64 first");
  rk::CellArgs a = {};
  a.x = d_x;
  a.out = d_out;
  a.ld_out = ld_out;
  a.n_series = n;
  a.kernels = b->d_cell;
  a.weights = esz == 8 ? (const void*)b->d_cw64 : (const void*)b->d_cw32;
  a.biases = esz == 8 ? (const void*)b->d_cb64 : (const void*)b->d_cb32;
  a.chidx = b->d_chidx;
  a.executed = d_exec;
  a.n_kernels = (int)b->K;
  a.l_series = b->L;
  a.n_channels = b->C;
  a.fpk = fpk;
  const size_t staged = (size_t)b->C * cell_sstride(b) * esz;
  if (!getenv("RK_NO_CELLROW")) {
    if (staged + 1024 <= st->smem_optin) {
      if (esz == 8)
        return fpk == 3 ? launch_cellrows<double, true, false>(b, st, a, stream, d_counters)
                        : launch_cellrows<double, false, false>(b, st, a, stream, d_counters);
      return launch_cellrows<float, true, false>(b, st, a, stream, d_counters);
    }
    if (esz == 8)
      return fpk == 3 ? launch_cellrows_gmem<double, true>(b, st, a, stream, d_counters)
                      : launch_cellrows_gmem<double, false>(b, st, a, stream, d_counters);
    return launch_cellrows_gmem<float, true>(b, st, a, stream, d_counters);
  }
  dim3 grid((unsigned)((b->K + 127) / 128), (unsigned)std::min<int64_t>(n, 65535));
  if (esz == 8) {
    if (fpk == 3)
      rk::rocket_cell_kernel<double, true><<<grid, 128, 0, stream>>>(a);
    else
      rk::rocket_cell_kernel<double, false><<<grid, 128, 0, stream>>>(a);
  } else {
    rk::rocket_cell_kernel<float, true><<<grid, 128, 0, stream>>>(a);
  }
  RK_CUDA(cudaGetLastError());
  return RK_OK;
}

int launch(rk_bank_t b, DeviceState* st, const void* d_xv, int64_t n, void* d_outv, int64_t ld_out, int fpk,
           int mode, cudaStream_t stream, unsigned long long* d_exec, int* d_counters, int esz) {
  if (n <= 0) return RK_OK;
  // float64, and MPV in exact mode (its ordered positive sum), run the cell
  // kernels; fast-mode MPV runs the wide kernels with summed positives
  if (esz == 8 || (fpk == 3 && (mode == RK_MODE_EXACT || !b->wide_path || b->gmem)))
    return launch_cells(b, st, d_xv, esz, n, d_outv, ld_out, fpk, stream, d_exec, d_counters);
  const float* d_x = static_cast<const float*>(d_xv);
  float* d_out = static_cast<float*>(d_outv);
  RK_CUDA(cudaMemsetAsync(d_counters, 0, sizeof(int) * kMaxLaunches, stream));
  if (b->wide_path) return launch_wide(b, st, d_x, n, d_out, ld_out, fpk, mode, stream, d_exec, d_counters);
  const int exact = mode == RK_MODE_EXACT ? 1 : 0;
  const int series_bytes = b->smem_bytes;
  // RK_PROFILE=1: time every class launch with events and report on stderr
  // (diagnostics only; serialises the host on each launch).
  static const bool profile = getenv("RK_PROFILE") != nullptr;
  std::vector<cudaEvent_t> prof_events;
  std::vector<int> prof_cls;
  std::vector<std::array<int, 4>> prof_info;
  const int smem_cap = (int)st->smem_optin - 1024;
  for (int cls = 0; cls < rk::kNumClasses; ++cls) {
    const int nchunks = b->cls_end[cls] - b->cls_begin[cls];
    if (nchunks <= 0) continue;
    KernelFn fn = kernel_table().fn[2 * exec_cls(cls, exact) + exact];
    // Stage several series per item when the class is too small to keep
    // all warps of a CTA busy on one series.
    int spi = 1;
    const int want = (4 * rk::kThreads / 32 + nchunks - 1) / nchunks;
    while (spi < want && spi < 16 && (int64_t)(spi + 1) * series_bytes <= smem_cap / 2 && spi < n) ++spi;
    const int smem = spi * series_bytes;
    int rc0 = set_kernel_smem(st, (const void*)fn, smem);
    if (rc0) return rc0;
    int ctas_per_sm = 1;
    RK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&ctas_per_sm, (const void*)fn, rk::kThreads, smem));
    ctas_per_sm = std::max(1, ctas_per_sm);
    const int64_t resident = (int64_t)st->sms * ctas_per_sm;
    const int64_t groups = (n + spi - 1) / spi;
    int nb = 1;
    while (nb < 64 && groups * nb < 4 * resident && nb * 2 <= nchunks / 8) nb *= 2;
    int* d_bs = nullptr;
    int rc = b->blocks_for(cls, nb, &d_bs);
    if (rc) return rc;
    rk::LaunchArgs a;
    a.x = d_x;
    a.out = d_out;
    a.ld_out = ld_out;
    a.n_items = groups * nb;
    a.n_series = n;
    a.chunks = b->d_chunks;
    a.weights = b->d_weights;
    a.chan_off = b->d_chan_off;
    a.block_start = d_bs;
    a.executed = d_exec;
    a.item_counter = d_counters + cls;
    a.n_blocks = nb;
    a.series_per_item = spi;
    a.n_channels = b->C;
    a.l_series = b->L;
    a.halo = b->halo;
    a.sstride = b->sstride;
    a.fpk = fpk;
    a.vec_out = (fpk == 2 && (ld_out % 2) == 0 && ((uintptr_t)d_out % 8) == 0) ? 1 : 0;
    a.vec_in = ((b->L % 4) == 0 && ((uintptr_t)d_x % 16) == 0 && (b->sstride % 4) == 0 && (b->halo % 4) == 0) ? 1 : 0;
    a.one = 1.0f;
    const int64_t grid = std::min<int64_t>(a.n_items, resident);
    if (profile) {
      cudaEvent_t e;
      cudaEventCreate(&e);
      cudaEventRecord(e, stream);
      prof_events.push_back(e);
      prof_cls.push_back(cls);
      prof_info.push_back({nchunks, spi, nb, (int)grid});
    }
    fn<<<(unsigned)grid, rk::kThreads, smem, stream>>>(a);
    RK_CUDA(cudaGetLastError());
  }
  if (profile && !prof_events.empty()) {
    // events between back-to-back launches (no host sync in between)
    cudaEvent_t e;
    cudaEventCreate(&e);
    cudaEventRecord(e, stream);
    prof_events.push_back(e);
    cudaEventSynchronize(e);
    for (size_t i = 0; i + 1 < prof_events.size(); ++i) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, prof_events[i], prof_events[i + 1]);
      const int cls = prof_cls[i];
      int64_t flops = 0;
      for (int k = b->cls_begin[cls]; k < b->cls_end[cls]; ++k) {
        const rk::DevChunk& c = b->chunks[k].dev;
        flops += (int64_t)2 * c.nk * c.nc * c.len * c.n;
      }
      fprintf(stderr,
              "RK_PROFILE class len=%d R=%d nck=%d exact=%d chunks=%d spi=%d nb=%d grid=%d ms=%.3f dense_tflops=%.2f\n",
              c_len(cls), rk::r_of((cls / rk::kNumNck) % rk::kNumR), cls % rk::kNumNck, exact, prof_info[i][0],
              prof_info[i][1], prof_info[i][2], prof_info[i][3], ms, flops * (double)n / (ms * 1e-3) / 1e12);
    }
    for (auto ev : prof_events) cudaEventDestroy(ev);
  }
  return RK_OK;
}

}  // namespace

extern "C" {

int rk_abi_version(void) { return RK_ABI_VERSION; }

// shared with the streaming runtime (rocket_stream.cu)
int rk_set_error(int code, const char* message) { return fail(code, "%s", message); }

// The device counter rk_transform accumulates executed positions into for
// device-pointer calls on `stream` (rk_internal.h).
int rk_stream_counter(rk_bank_t b, void* stream, unsigned long long** counter) {
  DeviceState* st = nullptr;
  int rc = device_state(b->device, &st);
  if (rc) return rc;
  return stream_scratch(st, stream ? (cudaStream_t)stream : st->stream, counter);
}

const char* rk_last_error(void) { return g_last_error.c_str(); }

int rk_device_count(int32_t* count) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    n = 0;
  }
  if (count) *count = n;
  return RK_OK;
}

namespace {
// half_margin (percent): a chunk runs half-warp when its modelled cost is
// below half_margin % of the best full-warp option; 0 builds the layout
// without lane-group chunks (the full-warp twin, rk_bank_s::narrow[0]);
// max_group caps the series per pass of the lane-group kinds (1 / 2 / 4 / 8).
int bank_create_impl(int64_t K, int32_t C, int32_t L, const int32_t* lengths, const int32_t* dilations,
                     const int32_t* paddings, const float* biases, const float* weights, const int64_t* woff,
                     const int32_t* chidx, const int64_t* choff, const int32_t* chcnt, int32_t device,
                     int64_t half_margin, int max_group, rk_bank_t* out) {
  if (!out) return fail(RK_ERR_INVALID, "bank output pointer is NULL");
  *out = nullptr;
  if (K < 1) return fail(RK_ERR_INVALID, "bank must contain at least one kernel");
  if (C < 1 || L < 1) return fail(RK_ERR_INVALID, "n_channels and l_series must be positive");
  if (K > (int64_t)1 << 30) return fail(RK_ERR_CAPACITY, "%lld kernels exceed the device bank limit", (long long)K);
  if (!lengths || !dilations || !paddings || !biases || !weights || !woff || !chidx || !choff || !chcnt)
    return fail(RK_ERR_INVALID, "bank array pointer is NULL");

  // ---- validate and key every kernel ----
  // Group key (dilation, lo, n, channel set): all kernels of a group share
  // the centre-position range [lo, lo + n) (lo = c*d - p, n = l_out), so
  // centred-padded kernels of every length share one group; shorter
  // kernels sit zero-padded inside a longer chunk (exact: zero taps add
  // +-0, which never changes the reference sum).
  struct Key {
    int d, lo, n;
    std::vector<int> ch;
    bool operator<(const Key& o) const { return std::tie(d, lo, n, ch) < std::tie(o.d, o.lo, o.n, o.ch); }
  };
  std::map<Key, std::vector<int64_t>> groups;
  int halo = 0;
  int64_t positions = 0, flops = 0;
  for (int64_t k = 0; k < K; ++k) {
    const int len = lengths[k], d = dilations[k], p = paddings[k], nc = chcnt[k];
    if (len < 0 || len > 11 || kLenIdx[len] < 0)
      return fail(RK_ERR_INVALID, "kernel %lld: length %d not in {7, 9, 11}", (long long)k, len);
    if (d < 1) return fail(RK_ERR_INVALID, "kernel %lld: dilation %d must be >= 1", (long long)k, d);
    if (p < 0) return fail(RK_ERR_INVALID, "kernel %lld: padding %d must be >= 0", (long long)k, p);
    const int64_t l_out = (int64_t)L + 2 * (int64_t)p - (int64_t)(len - 1) * d;
    if (l_out < 1)
      return fail(RK_ERR_INVALID, "kernel %lld: span %lld exceeds padded series length %lld", (long long)k,
                  (long long)(len - 1) * d, (long long)L + 2 * p);
    if ((int64_t)(len - 1) / 2 * d + L + p > (int64_t)1 << 30)
      return fail(RK_ERR_CAPACITY, "kernel %lld: dilation/padding too large", (long long)k);
    if (nc < 1 || nc > C) return fail(RK_ERR_INVALID, "kernel %lld: channel count %d out of range", (long long)k, nc);
    Key key{d, (len - 1) / 2 * d - p, (int)l_out, {}};
    for (int s = 0; s < nc; ++s) {
      const int ch = chidx[choff[k] + s];
      if (ch < 0 || ch >= C) return fail(RK_ERR_INVALID, "kernel %lld: channel index %d out of range", (long long)k, ch);
      key.ch.push_back(ch);
    }
    halo = std::max(halo, p);
    positions += l_out;
    // useful FLOPs: 2 per in-range tap + 1 bias add per output
    int64_t taps = 0;
    for (int j = 0; j < len; ++j) {
      // positions t in [0, l_out) with 0 <= t - p + j*d < L
      const int64_t off = (int64_t)j * d - p;
      const int64_t t_lo = std::max<int64_t>(0, -off), t_hi = std::min<int64_t>(l_out, (int64_t)L - off);
      if (t_hi > t_lo) taps += t_hi - t_lo;
    }
    flops += 2 * taps * nc + l_out;
    groups[key].push_back(k);
  }
  if (halo > (1 << 24)) return fail(RK_ERR_CAPACITY, "padding %d too large", halo);
  halo = (halo + 3) / 4 * 4;  // keep staged rows 16-byte aligned (float4 staging)

  DeviceState* st = nullptr;
  int rc = device_state(device, &st);
  if (rc) return rc;

  // Staged series: C channels of [halo zeros | L values | halo zeros],
  // stride rounded to 32 floats plus a pad e (a multiple of 4 floats: rows
  // stay 16-byte aligned for the bulk copies) chosen so that consecutive
  // staged series sit 16 banks apart (C * e = 16 mod 32): a half-warp
  // chunk's lanes 0-15 (series A) and 16-31 (series B) then read disjoint
  // bank halves instead of overlapping ones (r01: 55 % of the shared-load
  // wavefronts were bank-conflict replays at e = 4).
  int spad = 4;
  for (int e = 4; e < 32; e += 4)
    if ((C * e) % 32 == 16) {
      spad = e;
      break;
    }
  if (getenv("RK_SSTRIDE_PAD")) spad = std::max(4, atoi(getenv("RK_SSTRIDE_PAD")) / 4 * 4);
  int64_t sstride = (((int64_t)L + 2 * halo + 31) / 32) * 32 + spad;
  int64_t smem = (int64_t)C * sstride * 4;
  // A series that does not fit in shared memory is read from zero-haloed
  // rows in global memory instead (L1 / L2 resident; the wide kernel's
  // GMEM variants, run-time slot layout for every chunk).
  const bool gmem = smem > (int64_t)st->smem_optin - 1024;
  if (gmem && getenv("RK_NO_WIDE_PATH"))
    return fail(RK_ERR_CAPACITY,
                "one staged series needs %lld bytes of shared memory (C=%d, L=%d, halo=%d) but a CTA has %zu",
                (long long)smem, C, L, halo, st->smem_optin);

  std::unique_ptr<rk_bank_s> b(new rk_bank_s());
  b->device = device;
  b->gmem = gmem;
  b->K = K;
  b->C = C;
  b->L = L;
  b->halo = halo;
  b->sstride = (int)sstride;
  b->smem_bytes = (int)smem;
  b->n_groups = (int)groups.size();
  b->positions = positions;
  b->useful_flops = flops;

  // every chunk class runs on the wide kernel unless RK_NO_WIDE_PATH asks
  // for the class kernel (diagnostics)
  const bool wide_ok = !getenv("RK_NO_WIDE_PATH");
  // half-warp chunks: wide path, staged series; chosen when the cost model
  // says they beat the best full-warp R by the margin (percent, RK_HALF_MARGIN)
  // (and only when the wide path's CTAs can stage two series each at the
  // CTA count they will run at — launch_wide_chain's series-per-item rule —
  // otherwise items hold one series and the half classes would only run
  // their chunks on the full-warp kernel at an R priced for 16 lanes: 3
  // channels x L = 2048, 4 CTAs per SM, measured 0.4 % / 1.3 % slower)
  // CTAs per SM on the wide path (RK_WIDE_CTAS overrides): 3 x 8 warps, or
  // 2 x 12 for series of >= 32 KB staged (r02 sweeps, profiles/r02_cta_sweep.txt:
  // FordA shape +12 %, L = 2048 +2.6 %, config 5 +1.5 % against 6 x 4 and
  // 4 x 6; config 2 unchanged); 6 x 4 for series read from global memory
  // Small banks (< 2,000 kernels: few chunks per launch) keep narrower CTAs,
  // so no warp idles on an item (config 5 at 1k kernels: 2 x 12 was 4.5 %
  // slower than 4 x 6).
  const int cta_cap = getenv("RK_WIDE_CTAS") ? std::max(1, atoi(getenv("RK_WIDE_CTAS")))
                      : gmem || K < 2000     ? 6
                      : smem >= 32768        ? 2
                                             : 3;
  const int half_ctas = std::min<int>(
      std::min<int>(rk::kWideMaxWarps, (int)((st->smem_optin + 1024) / (smem + 1024))), cta_cap);
  const bool sp_ok = !getenv("RK_NO_SP");
  // RK_SP_RMAX: cap the positions per run of position-paired chunks (A/B)
  const int sp_rcap = getenv("RK_SP_RMAX") ? std::max(1, atoi(getenv("RK_SP_RMAX"))) : 15;
  // tail mode (chunks with fixed channel slots on the wide path): the cost
  // model may end a chunk's R-position runs at the last complete run and
  // walk the remaining positions one per lane instead of as partial runs
  const bool tail_ok = wide_ok && !gmem && !getenv("RK_NO_TAIL");
  const bool amap_ok = wide_ok && !gmem && !getenv("RK_NO_AMAP");
  const bool half_ok = half_margin > 0 && max_group >= 2 && wide_ok && !gmem && !getenv("RK_NO_HALF") &&
                       (int64_t)half_ctas * (2 * (int64_t)smem + 1024) <= (int64_t)st->smem_optin + 1024;
  // quarter-warp chunks (8 lanes per series, four series per pass): the
  // same rule with four staged series per CTA
  // margin of a quarter-warp option over the best so far (RK_QUARTER_MARGIN,
  // percent; default: the half-warp margin)
  const int64_t quarter_margin =
      getenv("RK_QUARTER_MARGIN") ? atoi(getenv("RK_QUARTER_MARGIN")) : half_margin;
  const bool quarter_ok = half_ok && max_group >= 4 && !getenv("RK_NO_QUARTER") &&
                          (int64_t)half_ctas * (4 * (int64_t)smem + 1024) <= (int64_t)st->smem_optin + 1024;
  // eighth-warp chunks (4 lanes per series, eight series per pass)
  const bool eighth_ok = quarter_ok && max_group >= 8 && !getenv("RK_NO_EIGHTH") &&
                         (int64_t)half_ctas * (8 * (int64_t)smem + 1024) <= (int64_t)st->smem_optin + 1024;
  const int64_t eighth_margin = getenv("RK_EIGHTH_MARGIN") ? atoi(getenv("RK_EIGHTH_MARGIN")) : quarter_margin;
  std::vector<float> wpack;
  std::vector<int> chan_off;
  for (auto& kv : groups) {
    const Key& key = kv.first;
    std::vector<int64_t> ks = kv.second;
    // longest kernels first: chunks are length-homogeneous except at the
    // boundaries between lengths
    std::stable_sort(ks.begin(), ks.end(), [&](int64_t x, int64_t y) { return lengths[x] > lengths[y]; });
    const int d = key.d, nc = (int)key.ch.size();
    const int n = key.n;
    size_t k0 = 0;
    while (k0 < ks.size()) {
      const size_t left = ks.size() - k0;
      // 1-channel groups: 4-kernel chunks (2 FFMA2 pairs), 1-pair chunks
      // for a remainder of 1 or 2; 2-channel groups: 1 pair per chunk (both
      // slots' weights in uniform registers); >= 3 channels: 1 pair per
      // chunk with the run-time slot loop (1 position per lane on the
      // class-kernel path).  Measured: 2 pairs with the slot loop (R <= 5
      // for registers) is slower both for 2 channels (-38 % at config 5) and
      // for 3+ (-17 % at C = 4).
      int P, nck;
      if (nc == 1) {
        P = left >= 3 ? 2 : 1;
        nck = P == 2 ? 0 : 3;
      } else {
        P = 1;
        nck = nc == 2 ? 1 : 2;
      }
      const int G = 2 * P;
      const int nk = (int)std::min<size_t>(G, left);
      const int len = lengths[ks[k0]];
      // a lone kernel runs position-paired (both FFMA2 lanes useful)
      const bool sp = nk == 1 && nc <= 2 && wide_ok && !gmem && sp_ok;
      if (sp) nck = nc == 1 ? 6 : 7;
      const int cc = (len - 1) / 2;
      HostChunk hc;
      std::memset(&hc.dev, 0, sizeof(hc.dev));
      rk::DevChunk& dc = hc.dev;
      dc.len = len;
      dc.d = d;
      dc.lo = key.lo;
      dc.n = n;
      dc.nk = nk;
      dc.nc = nc;
      dc.q32 = 32 / d;
      dc.r32 = 32 % d;
      dc.invd = 1.0f / (float)d;
      int best_r = 0;
      int64_t best = INT64_MAX;
      int lanes = 32;     // 16: half-warp, 8: quarter-warp, 4: eighth-warp chunk
      bool tail = false;  // complete runs at R, the remaining positions as an R = 1 map
      for (int ri = rk::kNumR - 1; ri >= 0; --ri) {
        if (sp) {
          // runs longer than 7 (9 at length 7) only pay on long position
          // ranges (measured: config 4 +1.2 %, L <= 2048 shapes -1 to -1.5 %)
          const int rlim = n >= 4096 ? rk::sp_rmax(nc, len) : std::min(rk::sp_rmax(nc, len), len == 7 ? 9 : 7);
          if (rk::r_of(ri) > std::min(rlim, sp_rcap)) continue;
          for (int tl = 0; tl < (tail_ok ? 2 : 1); ++tl) {
            const int64_t cst = chunk_cost_sp(len, d, n, nc, rk::r_of(ri), tl == 1);
            if (cst < best) {
              best = cst;
              best_r = ri;
              tail = tl == 1;
            }
          }
          continue;
        }
        if (nck == 2 && !wide_ok && ri != 0) continue;  // class-kernel generic path: 1 position per lane
        if (gmem && nck == 0 && ri > 2) continue;  // GMEM slot-loop kernels with 2 pairs: R <= 5 (registers)
        const bool fixed_slots = !gmem && rk::nck_slots(nck) != 0;
        for (int tl = 0; tl < (tail_ok && fixed_slots ? 2 : 1); ++tl) {
          const int64_t cst = chunk_cost(len, d, n, nc, P, rk::r_of(ri), !fixed_slots, 32, tl == 1);
          if (cst < best) {
            best = cst;
            best_r = ri;
            lanes = 32;
            tail = tl == 1;
          }
        }
        // single-channel chunks may run as half-warp chunks (two series per
        // pass of 16-lane steps: per series, half the 16-lane step cost) or
        // quarter-warp chunks (four series per pass of 8-lane steps)
        if (half_ok && nc == 1) {
          const int64_t fixed = 40 * 2 * P + 60;
          for (int tl = 0; tl < (tail_ok ? 2 : 1); ++tl) {
            const bool t = tl == 1;
            const int64_t c16 = (chunk_cost(len, d, n, nc, P, rk::r_of(ri), false, 16, t) - fixed) / 2 + fixed;
            if (c16 * 100 < best * half_margin) {
              best = c16;
              best_r = ri;
              lanes = 16;
              tail = t;
            }
            if (quarter_ok) {
              const int64_t c8 = (chunk_cost(len, d, n, nc, P, rk::r_of(ri), false, 8, t) - fixed) / 4 + fixed;
              if (c8 * 100 < best * quarter_margin) {
                best = c8;
                best_r = ri;
                lanes = 8;
                tail = t;
              }
            }
            if (eighth_ok) {
              const int64_t c4 = (chunk_cost(len, d, n, nc, P, rk::r_of(ri), false, 4, t) - fixed) / 8 + fixed;
              if (c4 * 100 < best * eighth_margin) {
                best = c4;
                best_r = ri;
                lanes = 4;
                tail = t;
              }
            }
          }
        }
      }
      if (lanes == 16) nck = nck == 0 ? 4 : 5;
      if (lanes == 8) nck = nck == 0 ? 8 : 9;
      if (lanes == 4) nck = nck == 0 ? 10 : 11;
      hc.cost = best;
      hc.tail = tail;
      // lane map: run-major where it replays fewer shared-memory wavefronts
      // (staged series, fixed channel slots; GMEM rows keep the residue-major
      // map, whose consecutive lanes read consecutive addresses)
      if (amap_ok && !sp && rk::nck_slots(nck) != 0 && rk::r_of(best_r) > 1) {
        int kg = 0;
        while (kg < 5 && (1 << (kg + 1)) <= lanes && d % (1 << (kg + 1)) == 0) ++kg;
        const int R = rk::r_of(best_r);
        const int64_t w_res = lanemap_wavefronts(d, n, R, lanes, -1);
        const int64_t w_run = lanemap_wavefronts(d, n, R, lanes, kg);
        if (w_run < w_res) hc.amap = kg;
      }
      dc.cls = (kLenIdx[len] * rk::kNumR + best_r) * rk::kNumNck + nck;
      // weights: [slot][pair][tap][2]; a shorter kernel (ck < cc) is
      // centred in the LEN-tap frame with zero taps at both ends.
      while (wpack.size() % 4) wpack.push_back(0.0f);
      dc.wofs = (int)wpack.size();
      for (int s = 0; s < nc; ++s)
        for (int pp = 0; pp < P; ++pp)
          for (int j = 0; j < len; ++j)
            for (int h = 0; h < 2; ++h) {
              const int g = 2 * pp + h;
              float w = 0.0f;
              if (sp) {
                // position-paired: the one kernel's weight in both lanes (w, w)
                const int64_t k = ks[k0];
                const int lk = lengths[k], ck = (lk - 1) / 2;
                const int jj = j - (cc - ck);
                if (jj >= 0 && jj < lk) w = weights[woff[k] + (int64_t)s * lk + jj];
              } else if (g < nk) {
                const int64_t k = ks[k0 + g];
                const int lk = lengths[k], ck = (lk - 1) / 2;
                const int jj = j - (cc - ck);
                if (jj >= 0 && jj < lk) w = weights[woff[k] + (int64_t)s * lk + jj];
              }
              wpack.push_back(w);
            }
      dc.chofs = (int)chan_off.size();
      for (int s = 0; s < nc; ++s) chan_off.push_back(key.ch[s] * (int)sstride);
      for (int g = 0; g < 4; ++g) {
        if (g < nk) {
          const int64_t k = ks[k0 + g];
          // -0.0 -> +0.0: identical results for the reference (acc is never -0),
          // and keeps the fast path's accumulator init sign-clean.
          const float bias = biases[k] + 0.0f;
          dc.col[g] = (int)k;
          dc.bias[g] = bias;
        } else {
          dc.col[g] = -1;
          dc.bias[g] = 0.0f;
        }
      }
      b->chunks.push_back(hc);
      k0 += nk;
    }
  }
  for (const auto& hc : b->chunks) b->max_groups = std::max(b->max_groups, rk::nck_groups(hc.dev.cls % rk::kNumNck));
  // Row pad by the lane-group mix: consecutive staged series sit C*e banks
  // apart and a group of LG lanes reads LG consecutive banks, so pick the
  // pad e whose group offsets overlap least, weighted by the modelled cost
  // of each group width (eighth-warp chunks want 4 banks, quarter 8, half 16;
  // at e = 16 eight 4-lane groups met in two bank ranges: 4-way replays).
  if (!getenv("RK_SSTRIDE_PAD") && b->max_groups > 1 && !gmem) {
    int64_t wcost[4] = {0, 0, 0, 0};  // by log2(groups): 1, 2, 4, 8
    for (const auto& hc : b->chunks) {
      const int g = rk::nck_groups(hc.dev.cls % rk::kNumNck);
      wcost[g == 8 ? 3 : g == 4 ? 2 : g == 2 ? 1 : 0] += hc.cost;
    }
    int best_e = spad;
    double best_score = 1e300;
    for (int e = 4; e < 32; e += 4) {
      double score = (double)wcost[0];
      for (int j = 1; j < 4; ++j) {
        const int groups = 1 << j, lg = 32 / groups;
        int cover[32] = {};
        for (int g = 0; g < groups; ++g)
          for (int l = 0; l < lg; ++l) ++cover[(g * C * e + l) % 32];
        int mult = 1;
        for (int k2 = 0; k2 < 32; ++k2) mult = std::max(mult, cover[k2]);
        score += (double)wcost[j] * mult;
      }
      if (score < best_score) {
        best_score = score;
        best_e = e;
      }
    }
    if (best_e != spad) {
      const int64_t old_stride = sstride;
      sstride = (((int64_t)L + 2 * halo + 31) / 32) * 32 + best_e;
      smem = (int64_t)C * sstride * 4;
      for (auto& o : chan_off) o = (int)(o / old_stride * sstride);
      b->sstride = (int)sstride;
      b->smem_bytes = (int)smem;
    }
  }
  // RK_DUMP_CHUNKS=<path>: the chunk layout, one line per chunk (diagnostics)
  if (const char* dump = getenv("RK_DUMP_CHUNKS")) {
    if (FILE* f = fopen(dump, "a")) {
      fprintf(f, "# bank K=%lld C=%d L=%d half_margin=%lld\n", (long long)K, C, L, (long long)half_margin);
      for (const auto& hc : b->chunks) {
        const rk::DevChunk& c = hc.dev;
        fprintf(f, "len=%d R=%d nck=%d d=%d lo=%d n=%d nk=%d nc=%d cost=%lld tail=%d amap=%d\n", c.len,
                rk::r_of((c.cls / rk::kNumNck) % rk::kNumR), c.cls % rk::kNumNck, c.d, c.lo, c.n, c.nk, c.nc,
                (long long)hc.cost, hc.tail ? 1 : 0, hc.amap);
      }
      fclose(f);
    }
  }
  // Both modes accumulate the taps without the bias and count acc > -bias
  // (RN(acc + b) > 0 <=> acc > -b exactly); "+ 0.0f" keeps the threshold
  // off -0 (the kernel's compare is a plain setp.gt).
  for (auto& hc : b->chunks)
    for (int g = 0; g < 4; ++g) hc.dev.thr[g] = -hc.dev.bias[g] + 0.0f;
  // class-major order (keeps the warps of a CTA in one code path), then
  // descending cost (long chunks first, short ones fill the tail).
  std::stable_sort(b->chunks.begin(), b->chunks.end(), [](const HostChunk& x, const HostChunk& y) {
    if (x.dev.cls != y.dev.cls) return x.dev.cls < y.dev.cls;
    return x.cost > y.cost;
  });
  for (int c = 0; c < rk::kNumClasses; ++c) b->cls_begin[c] = b->cls_end[c] = 0;
  for (size_t i = 0; i < b->chunks.size(); ++i) {
    const int c = b->chunks[i].dev.cls;
    if (i == 0 || b->chunks[i - 1].dev.cls != c) b->cls_begin[c] = (int)i;
    b->cls_end[c] = (int)i + 1;
  }
  b->cost_prefix.assign(b->chunks.size() + 1, 0);
  for (size_t i = 0; i < b->chunks.size(); ++i) b->cost_prefix[i + 1] = b->cost_prefix[i] + b->chunks[i].cost;

  // Wide path (every bank; fixed slots for 1-2 channels, the run-time slot
  // loop beyond).  CTAs per SM as shared memory allows, at most cta_cap;
  // warps per CTA so the SM holds 24 warps (the ~80-register budget).
  {
    const int per_cta = (gmem ? 0 : (int)smem) + 1024;  // + the per-CTA reservation
    const int by_smem = std::min<int>(rk::kWideMaxWarps, (int)((st->smem_optin + 1024) / per_cta));
    const int cap = cta_cap;
    if (by_smem >= 1 && wide_ok) {
      b->wide_path = true;
      b->wide_ctas_smem = by_smem;
      b->wide_ctas_per_sm = std::min(by_smem, cap);
      const int blob_bytes = rk::kBlobFloat4 * 16;
      for (int cls = 0; cls < rk::kNumClasses; ++cls) {
        const int cb = b->cls_begin[cls], ce = b->cls_end[cls];
        if (ce <= cb) continue;
        const int nck = cls % rk::kNumNck;
        const int P = rk::nck_pairs(nck), NC = gmem ? 0 : rk::nck_slots(nck);
        const int len = 7 + 2 * (cls / (rk::kNumNck * rk::kNumR));
        // bytes after the descriptor: fixed slots -> the weights; run-time
        // slots -> the weights then the slot list (16-byte aligned)
        auto data_bytes = [&](const rk::DevChunk& c) {
          return NC ? NC * P * len * 8 : c.nc * P * len * 8 + ((c.nc * 4 + 15) / 16) * 16;
        };
        int i0 = cb;
        while (i0 < ce) {
          int nch = 0, used = 0;
          while (i0 + nch < ce) {
            const int add = (int)sizeof(rk::WChunk) + data_bytes(b->chunks[i0 + nch].dev);
            if (used + add > blob_bytes) break;
            used += add;
            ++nch;
          }
          if (nch == 0) return fail(RK_ERR_CAPACITY, "a chunk's weights exceed the kernel parameter block");
          rk_bank_s::WideLaunch wl;
          wl.cls = cls;
          wl.n_chunks = nch;
          wl.dense_flops = 0;
          wl.blob.assign(rk::kBlobFloat4, rk::float4_t{0, 0, 0, 0});
          char* raw = reinterpret_cast<char*>(wl.blob.data());
          std::vector<std::pair<int, int>> wranges;  // float ranges holding weights (negated for fast mode)
          int cursor = nch * (int)sizeof(rk::WChunk);
          for (int j = 0; j < nch; ++j) {
            const rk::DevChunk& c = b->chunks[i0 + j].dev;
            rk::WChunk wc;
            std::memset(&wc, 0, sizeof(wc));
            wc.d = c.d;
            wc.lo = c.lo;
            wc.n = c.n;
            wc.nk = c.nk;
            for (int g = 0; g < 4; ++g) {
              wc.col[g] = c.col[g];
              wc.bias[g] = c.bias[g];
              wc.thr[g] = c.thr[g];
            }
            const int wbytes = c.nc * P * len * 8;
            if (NC) {
              for (int s2 = 0; s2 < NC; ++s2) wc.ch[s2] = chan_off[c.chofs + s2] / (int)sstride;
            } else {
              wc.ch[0] = cursor;
              wc.ch[1] = c.nc;
            }
            wc.q32 = (short)c.q32;
            const HostChunk& hcj = b->chunks[i0 + j];
            wc.r32 = (short)(c.r32 | (hcj.tail ? rk::kTailFlag : 0) |
                             (hcj.amap >= 0 ? rk::kAMapFlag | (hcj.amap << 8) : 0));
            wc.invd = c.invd;
            std::memcpy(raw + (size_t)j * sizeof(rk::WChunk), &wc, sizeof(wc));
            std::memcpy(raw + cursor, wpack.data() + c.wofs, wbytes);
            wranges.emplace_back(cursor / 4, wbytes / 4);
            if (!NC) {
              int* slots = reinterpret_cast<int*>(raw + cursor + wbytes);
              for (int s2 = 0; s2 < c.nc; ++s2) slots[s2] = chan_off[c.chofs + s2] / (int)sstride;
            }
            cursor += data_bytes(c);
            wl.dense_flops += (int64_t)2 * c.nk * c.nc * c.len * c.n;
          }
          // fast mode computes acc' = -b + sum (-w) x; (-w) * x == w * (-x)
          // bit for bit, so negating the weights replaces negating the
          // staged series and lets the rows be bulk-copied unchanged
          wl.blob_fast = wl.blob;
          float* wf = reinterpret_cast<float*>(wl.blob_fast.data());
          for (const auto& r : wranges)
            for (int q = 0; q < r.second; ++q) wf[r.first + q] = -wf[r.first + q];
          b->wide_launches.push_back(std::move(wl));
          i0 += nch;
        }
      }
      if ((int)b->wide_launches.size() > kMaxLaunches) {
        b->wide_path = false;
        b->wide_launches.clear();
      }
    }
  }

  std::vector<rk::DevChunk> dev(b->chunks.size());
  for (size_t i = 0; i < b->chunks.size(); ++i) dev[i] = b->chunks[i].dev;
  if (wpack.empty()) wpack.push_back(0.0f);
  RK_CUDA(cudaSetDevice(device));
  RK_CUDA(cudaMalloc(&b->d_chunks, sizeof(rk::DevChunk) * dev.size()));
  RK_CUDA(cudaMalloc(&b->d_weights, sizeof(float) * wpack.size()));
  RK_CUDA(cudaMalloc(&b->d_chan_off, sizeof(int) * chan_off.size()));
  RK_CUDA(cudaMemcpy(b->d_chunks, dev.data(), sizeof(rk::DevChunk) * dev.size(), cudaMemcpyHostToDevice));
  RK_CUDA(cudaMemcpy(b->d_weights, wpack.data(), sizeof(float) * wpack.size(), cudaMemcpyHostToDevice));
  RK_CUDA(cudaMemcpy(b->d_chan_off, chan_off.data(), sizeof(int) * chan_off.size(), cudaMemcpyHostToDevice));
  // cell path: kernels sorted by (len*nc, l_out) so warp neighbours share
  // trip counts; weights in the reference layout
  {
    int64_t nw = 0, nci = 0;
    for (int64_t k = 0; k < K; ++k) {
      nw = std::max<int64_t>(nw, woff[k] + (int64_t)lengths[k] * chcnt[k]);
      nci = std::max<int64_t>(nci, choff[k] + chcnt[k]);
    }
    b->n_weights = nw;
    b->cell_order.resize(K);
    for (int64_t k = 0; k < K; ++k) b->cell_order[k] = k;
    auto l_out_of = [&](int64_t k) { return (int64_t)L + 2 * paddings[k] - (int64_t)(lengths[k] - 1) * dilations[k]; };
    // (length, channels, padded?, dilation, padding): a warp of the staged
    // cell kernel gets one length and mostly one (d, p), so its lanes read
    // the same shared-memory words, and unpadded kernels (l_out = L - (len-1)d)
    // are kept apart from centred ones (l_out = L), so a warp's trip count
    // (its longest l_out) wastes few lane slots: 0.90 -> 0.985 of the lane
    // slots useful at L = 1024
    std::stable_sort(b->cell_order.begin(), b->cell_order.end(), [&](int64_t x, int64_t y) {
      return std::make_tuple(lengths[x], chcnt[x], paddings[x] > 0, dilations[x], paddings[x]) <
             std::make_tuple(lengths[y], chcnt[y], paddings[y] > 0, dilations[y], paddings[y]);
    });
    for (int li = 0; li < 3; ++li) {
      b->cell_len_begin[li] = b->cell_len_end[li] = 0;
    }
    for (int64_t i = 0; i < K; ++i) {
      const int li = kLenIdx[lengths[b->cell_order[i]]];
      if (i == 0 || kLenIdx[lengths[b->cell_order[i - 1]]] != li) b->cell_len_begin[li] = i;
      b->cell_len_end[li] = i + 1;
    }
    std::vector<rk::CellKernel> ck(K);
    std::vector<float> cb(K);
    for (int64_t i = 0; i < K; ++i) {
      const int64_t k = b->cell_order[i];
      ck[i] = rk::CellKernel{lengths[k], dilations[k], paddings[k], chcnt[k], (int)l_out_of(k), (int)woff[k],
                             (int)choff[k], (int)k};
      cb[i] = biases[k];
    }
    RK_CUDA(cudaMalloc(&b->d_cell, sizeof(rk::CellKernel) * K));
    RK_CUDA(cudaMalloc(&b->d_chidx, sizeof(int) * std::max<int64_t>(1, nci)));
    RK_CUDA(cudaMalloc(&b->d_cw32, sizeof(float) * std::max<int64_t>(1, nw)));
    RK_CUDA(cudaMalloc(&b->d_cb32, sizeof(float) * K));
    RK_CUDA(cudaMemcpy(b->d_cell, ck.data(), sizeof(rk::CellKernel) * K, cudaMemcpyHostToDevice));
    RK_CUDA(cudaMemcpy(b->d_chidx, chidx, sizeof(int) * nci, cudaMemcpyHostToDevice));
    RK_CUDA(cudaMemcpy(b->d_cw32, weights, sizeof(float) * nw, cudaMemcpyHostToDevice));
    RK_CUDA(cudaMemcpy(b->d_cb32, cb.data(), sizeof(float) * K, cudaMemcpyHostToDevice));
  }
  b->device_bytes = (int64_t)(sizeof(rk::DevChunk) * dev.size() + sizeof(float) * wpack.size() +
                              sizeof(int) * chan_off.size());
  *out = b.release();
  return RK_OK;
}
}  // namespace

int rk_bank_create(int64_t K, int32_t C, int32_t L, const int32_t* lengths, const int32_t* dilations,
                   const int32_t* paddings, const float* biases, const float* weights,
                   const int64_t* woff, const int32_t* chidx, const int64_t* choff, const int32_t* chcnt,
                   int32_t device, rk_bank_t* out) {
  // the half-warp margin of the cost model, per mode (measured optima:
  // profiles/r01_half_margin_sweep.txt)
  const int64_t margin_fast = getenv("RK_HALF_MARGIN") ? atoi(getenv("RK_HALF_MARGIN")) : 101;
  // (exact: 103 after the run-major map and eighth-warp chunks; the sweep
  // 103 / 105 / 107 / 110 is in profiles/r02_cta_sweep.txt)
  const int64_t margin_exact = getenv("RK_HALF_MARGIN_EXACT") ? atoi(getenv("RK_HALF_MARGIN_EXACT")) : 103;
  int rc = bank_create_impl(K, C, L, lengths, dilations, paddings, biases, weights, woff, chidx, choff, chcnt, device,
                            margin_fast, 8, out);
  if (rc) return rc;
  rk_bank_t b = *out;
  auto impl = [&](int64_t margin, int max_group, rk_bank_t* dst) -> int {
    int r = bank_create_impl(K, C, L, lengths, dilations, paddings, biases, weights, woff, chidx, choff, chcnt,
                             device, margin, max_group, dst);
    if (r) {
      delete b;
      *out = nullptr;
      return r;
    }
    b->device_bytes += (*dst)->device_bytes;
    return RK_OK;
  };
  // Narrower twins for items that cannot fill this layout's widest lane
  // groups: e.g. the config-2 bank at 2,000 series (one series per item)
  // runs the full-warp twin (-6 % fast, -11 % exact otherwise).
  auto narrow_twins = [&](rk_bank_t x, int64_t margin, int from) -> int {
    for (int j = from; j < 3; ++j) {
      const int g = 1 << j;
      if (g >= x->max_groups) break;
      int r = impl(g == 1 ? 0 : margin, g, &x->narrow[j]);
      if (r) return r;
    }
    return RK_OK;
  };
  if ((rc = narrow_twins(b, margin_fast, 0))) return rc;
  // exact mode (FMUL2 + FFMA2 per tap) favours lane groups more: its own
  // layout priced with margin_exact (FordA shape exact 330k -> 354k with
  // quarter-warp chunks), with its own narrower twins (items of one series
  // run the fast layout's full-warp twin, which is mode-independent)
  if (margin_exact != margin_fast && b->max_groups > 1) {
    if ((rc = impl(margin_exact, 8, &b->exact_bank))) return rc;
    if (b->exact_bank->max_groups == 1) {
      b->device_bytes -= b->exact_bank->device_bytes;
      delete b->exact_bank;
      b->exact_bank = nullptr;
    } else if ((rc = narrow_twins(b->exact_bank, margin_exact, 1))) {
      return rc;
    }
  }
  return RK_OK;
}

int rk_bank_destroy(rk_bank_t bank) {
  delete bank;
  return RK_OK;
}

int rk_bank_info(rk_bank_t b, rk_bank_info_t* info) {
  if (!b || !info) return fail(RK_ERR_INVALID, "NULL bank or info");
  std::memset(info, 0, sizeof(*info));
  info->n_kernels = b->K;
  info->n_channels = b->C;
  info->l_series = b->L;
  info->n_groups = b->n_groups;
  info->n_chunks = (int32_t)b->chunks.size();
  info->halo = b->halo;
  info->smem_bytes = b->smem_bytes;
  info->positions_per_series = b->positions;
  info->useful_flops_per_series = b->useful_flops;
  info->device_bytes = b->device_bytes;
  info->device = b->device;
  info->path = b->wide_path ? (b->gmem ? 2 : 1) : 0;
  info->ctas_per_sm = b->wide_ctas_per_sm;
  for (const auto& hc : b->chunks) {
    info->n_half_chunks += rk::nck_half(hc.dev.cls % rk::kNumNck) ? 1 : 0;
    info->n_quarter_chunks += rk::nck_quarter(hc.dev.cls % rk::kNumNck) ? 1 : 0;
    info->n_eighth_chunks += rk::nck_eighth(hc.dev.cls % rk::kNumNck) ? 1 : 0;
    info->n_paired_chunks += rk::nck_sp(hc.dev.cls % rk::kNumNck) ? 1 : 0;
    info->n_runmajor_chunks += hc.amap >= 0 ? 1 : 0;
  }
  if (b->wide_path)
    info->n_launches = (int32_t)b->wide_launches.size();
  else
    for (int c = 0; c < rk::kNumClasses; ++c) info->n_launches += b->cls_end[c] > b->cls_begin[c] ? 1 : 0;
  return RK_OK;
}

int rk_transform(rk_bank_t b, const void* xv, int32_t dtype, int64_t n, void* outv, int64_t ld_out, int64_t row0,
                 int32_t fpk, int32_t mode, void* stream_ptr, int64_t* executed) {
  RkRange range("rk_transform n=%lld mode=%lld", (long long)n, (long long)mode);
  if (!b) return fail(RK_ERR_INVALID, "NULL bank");
  if (n < 0 || row0 < 0) return fail(RK_ERR_INVALID, "n_series and row0 must be non-negative");
  if (fpk != 2 && fpk != 3) return fail(RK_ERR_INVALID, "features_per_kernel=%d must be 2 or 3", fpk);
  if (dtype != RK_DTYPE_F32 && dtype != RK_DTYPE_F64) return fail(RK_ERR_INVALID, "unknown dtype %d", dtype);
  const int esz = dtype == RK_DTYPE_F64 ? 8 : 4;
  const char* x = static_cast<const char*>(xv);
  char* out = static_cast<char*>(outv);
  if (mode != RK_MODE_EXACT && mode != RK_MODE_FAST) return fail(RK_ERR_INVALID, "unknown mode %d", mode);
  if (ld_out < b->K * fpk) return fail(RK_ERR_INVALID, "ld_out %lld < n_kernels * fpk", (long long)ld_out);
  if (executed) *executed = 0;
  if (n == 0) return RK_OK;
  if (!x || !out) return fail(RK_ERR_INVALID, "NULL x or out");
  DeviceState* st = nullptr;
  int rc = device_state(b->device, &st);
  if (rc) return rc;
  RK_CUDA(cudaSetDevice(b->device));
  const bool dx = is_device_pointer(x), dout = is_device_pointer(out);
  const int64_t row_in = (int64_t)b->C * b->L;
  if (dx && dout) {
    // Device-resident: asynchronous on the caller's stream (or the
    // library's); the counters live in that stream's scratch block.  A NULL
    // stream means the caller's default (legacy) stream: the library stream
    // is non-blocking, so it waits for the work already queued there (e.g.
    // the H2D copy of x) and the default stream waits for the transform.
    cudaStream_t stream = stream_ptr ? (cudaStream_t)stream_ptr : st->stream;
    cudaEvent_t ev_in = nullptr;
    if (!stream_ptr) {
      RK_CUDA(cudaEventCreateWithFlags(&ev_in, cudaEventDisableTiming));
      RK_CUDA(cudaEventRecord(ev_in, (cudaStream_t)0));
      RK_CUDA(cudaStreamWaitEvent(stream, ev_in, 0));
      RK_CUDA(cudaEventDestroy(ev_in));
    }
    std::mutex* smu = nullptr;
    {
      std::lock_guard<std::mutex> lk(st->pool_mu);
      auto& m = st->stream_mu[stream];
      if (!m) m.reset(new std::mutex());
      smu = m.get();
    }
    std::lock_guard<std::mutex> stream_lock(*smu);
    unsigned long long* d_exec = nullptr;
    rc = stream_scratch(st, stream, &d_exec);
    if (rc) return rc;
    RK_CUDA(cudaMemsetAsync(d_exec, 0, sizeof(unsigned long long), stream));
    rc = launch(b, st, x, n, out + row0 * ld_out * esz, ld_out, fpk, mode, stream, d_exec,
                reinterpret_cast<int*>(d_exec + 1), esz);
    if (rc) return rc;
    if (!stream_ptr) {
      cudaEvent_t ev_out = nullptr;
      RK_CUDA(cudaEventCreateWithFlags(&ev_out, cudaEventDisableTiming));
      RK_CUDA(cudaEventRecord(ev_out, stream));
      RK_CUDA(cudaStreamWaitEvent((cudaStream_t)0, ev_out, 0));
      RK_CUDA(cudaEventDestroy(ev_out));
    }
    if (executed) {
      unsigned long long h = 0;
      RK_CUDA(cudaMemcpyAsync(&h, d_exec, sizeof(h), cudaMemcpyDeviceToHost, stream));
      RK_CUDA(cudaStreamSynchronize(stream));
      *executed = (int64_t)h;
    }
    return RK_OK;
  }
  // Pageable host buffers (numpy arrays): the pinned-ring pipeline, whose
  // host copies run on several threads (the first touch of a fresh output
  // array is the bottleneck otherwise).
  if (!dx && !dout && (!is_pinned_host(x) || !is_pinned_host(out)) && !getenv("RK_NO_HOST_RING"))
    return rk_stream_host(b, x, dtype, n, out, ld_out, row0, fpk, mode, executed);
  // Pinned host buffers: row batches through a pooled worker's device
  // buffers on three streams (see Worker).
  Worker* w = nullptr;
  rc = acquire_worker(st, &w);
  if (rc) return rc;
  struct Release {
    DeviceState* st;
    Worker* w;
    ~Release() { release_worker(st, w); }
  } release{st, w};
  cudaStream_t stream = w->stream;
  const int64_t out_row_bytes = b->K * fpk * esz;
  const int64_t in_row_bytes = row_in * esz;
  const int64_t budget = (int64_t)1 << 30;  // device scratch per output buffer
  int64_t batch = std::max<int64_t>(1, budget / out_row_bytes);
  batch = std::min<int64_t>(batch, n);
  // several batches when there is enough work to overlap the copies
  const int64_t nbatch_min = getenv("RK_E2E_BATCHES") ? std::max(1, atoi(getenv("RK_E2E_BATCHES"))) : 6;
  const int64_t min_rows = getenv("RK_E2E_MIN_ROWS") ? std::max(1, atoi(getenv("RK_E2E_MIN_ROWS"))) : 4096;
  if (n >= min_rows) batch = std::min<int64_t>(batch, (n + nbatch_min - 1) / nbatch_min);
  // Few rows: up to three equal batches of >= 1,000 rows, so the features of
  // one batch copy out while the next computes (FordA shape, 3,601 rows: one
  // batch 311k -> three 413k series/s end to end; smaller batches turn
  // launch-bound: 8 batches 164k).
  else if (!getenv("RK_E2E_BATCHES"))
    batch = std::min<int64_t>(batch, (n + std::max<int64_t>(1, std::min<int64_t>(3, n / 1000)) - 1) /
                                         std::max<int64_t>(1, std::min<int64_t>(3, n / 1000)));
  // Batch schedule: the features of a batch are complete only when its whole
  // launch chain has run, so the last batch's D2H is exposed after the last
  // kernel.  Batches shrink geometrically towards the end (tail rows, x2
  // backwards up to `batch`): at config 2 the exposed copy drops from
  // 1.33 GB (27 ms) to 0.33 GB.
  std::vector<int64_t> sizes;
  {
    const int64_t tail_min = getenv("RK_E2E_TAIL") ? std::max(1, atoi(getenv("RK_E2E_TAIL"))) : 4096;
    int64_t rem = n, sz = n >= min_rows ? std::min<int64_t>(batch, std::max<int64_t>(tail_min, n / 32)) : batch;
    while (rem > 0) {
      const int64_t take = std::min(sz, rem);
      sizes.push_back(take);
      rem -= take;
      sz = std::min<int64_t>(2 * sz, batch);
    }
    std::reverse(sizes.begin(), sizes.end());
  }
  std::vector<int64_t> starts(sizes.size() + 1, 0);
  for (size_t k = 0; k < sizes.size(); ++k) starts[k + 1] = starts[k] + sizes[k];
  if (!dx) {
    const size_t need = (size_t)(batch * in_row_bytes);
    if (need > w->in_cap) {
      for (int i = 0; i < kInBufs; ++i) {
        if (w->d_in[i]) RK_CUDA(cudaFree(w->d_in[i]));
        w->d_in[i] = nullptr;
        RK_CUDA(cudaMalloc(&w->d_in[i], need));
      }
      w->in_cap = need;
    }
  }
  if (!dout) {
    const size_t need = (size_t)(batch * out_row_bytes);
    if (need > w->out_cap) {
      for (int i = 0; i < kOutBufs; ++i) {
        if (w->d_out[i]) RK_CUDA(cudaFree(w->d_out[i]));
        w->d_out[i] = nullptr;
        RK_CUDA(cudaMalloc(&w->d_out[i], need));
      }
      w->out_cap = need;
    }
  }
  unsigned long long* d_exec = w->d_scratch;
  RK_CUDA(cudaMemsetAsync(d_exec, 0, sizeof(unsigned long long), stream));
  const int64_t nbatch = (int64_t)sizes.size();
  auto h2d = [&](int64_t k) -> int {
    const int64_t s0 = starts[k], cnt = sizes[k];
    const int ib = (int)(k % kInBufs);
    if (k >= kInBufs) RK_CUDA(cudaStreamWaitEvent(w->h2d_stream, w->in_free[ib], 0));
    RK_CUDA(cudaMemcpyAsync(w->d_in[ib], x + s0 * in_row_bytes, cnt * in_row_bytes, cudaMemcpyHostToDevice,
                            w->h2d_stream));
    RK_CUDA(cudaEventRecord(w->in_ready[ib], w->h2d_stream));
    return RK_OK;
  };
  if (!dx) {
    rc = h2d(0);
    if (rc) return rc;
  }
  for (int64_t k = 0; k < nbatch; ++k) {
    const int64_t s0 = starts[k], cnt = sizes[k];
    const int ib = (int)(k % kInBufs), ob = (int)(k % kOutBufs);
    RkRange brange("rk pinned batch %lld rows=%lld", (long long)k, (long long)cnt);
    if (!dx && k + 1 < nbatch) {
      rc = h2d(k + 1);  // enqueued before this batch's D2H
      if (rc) return rc;
    }
    const void* kx = x + s0 * in_row_bytes;
    if (!dx) {
      RK_CUDA(cudaStreamWaitEvent(stream, w->in_ready[ib], 0));
      kx = w->d_in[ib];
    }
    void* ko = dout ? (void*)(out + (row0 + s0) * ld_out * esz) : (void*)w->d_out[ob];
    const int64_t kld = dout ? ld_out : b->K * fpk;
    if (!dout && k >= kOutBufs) RK_CUDA(cudaStreamWaitEvent(stream, w->out_free[ob], 0));
    rc = launch(b, st, kx, cnt, ko, kld, fpk, mode, stream, d_exec, reinterpret_cast<int*>(d_exec + 1), esz);
    if (rc) return rc;
    if (!dx) RK_CUDA(cudaEventRecord(w->in_free[ib], stream));
    if (!dout) {
      RK_CUDA(cudaEventRecord(w->out_ready[ob], stream));
      RK_CUDA(cudaStreamWaitEvent(w->d2h_stream, w->out_ready[ob], 0));
      char* hdst = out + (row0 + s0) * ld_out * esz;
      if (ld_out == kld) {
        RK_CUDA(cudaMemcpyAsync(hdst, w->d_out[ob], cnt * out_row_bytes, cudaMemcpyDeviceToHost, w->d2h_stream));
      } else {
        RK_CUDA(cudaMemcpy2DAsync(hdst, ld_out * esz, w->d_out[ob], kld * esz, kld * esz, cnt, cudaMemcpyDeviceToHost,
                                  w->d2h_stream));
      }
      RK_CUDA(cudaEventRecord(w->out_free[ob], w->d2h_stream));
    }
  }
  unsigned long long h = 0;
  RK_CUDA(cudaMemcpyAsync(&h, d_exec, sizeof(h), cudaMemcpyDeviceToHost, stream));
  RK_CUDA(cudaStreamSynchronize(w->d2h_stream));
  RK_CUDA(cudaStreamSynchronize(w->h2d_stream));
  RK_CUDA(cudaStreamSynchronize(stream));
  if (executed) *executed = (int64_t)h;
  return RK_OK;
}

int rk_transform_f32(rk_bank_t b, const float* x, int64_t n, float* out, int64_t ld_out, int64_t row0,
                     int32_t fpk, int32_t mode, void* stream, int64_t* executed) {
  return rk_transform(b, x, RK_DTYPE_F32, n, out, ld_out, row0, fpk, mode, stream, executed);
}

int rk_bank_attach_f64(rk_bank_t b, const double* biases, const double* weights) {
  if (!b || !biases || !weights) return fail(RK_ERR_INVALID, "NULL bank or array");
  RK_CUDA(cudaSetDevice(b->device));
  std::vector<double> cb(b->K);
  for (int64_t i = 0; i < b->K; ++i) cb[i] = biases[b->cell_order[i]];
  // one attach at a time per bank; a transform sees the parameters only
  // once they are complete (f64_ready)
  std::lock_guard<std::mutex> lk(b->mu);
  if (b->f64_ready.load(std::memory_order_acquire)) return RK_OK;  // immutable bank: attached once
  if (!b->d_cw64) RK_CUDA(cudaMalloc(&b->d_cw64, sizeof(double) * std::max<int64_t>(1, b->n_weights)));
  if (!b->d_cb64) RK_CUDA(cudaMalloc(&b->d_cb64, sizeof(double) * b->K));
  RK_CUDA(cudaMemcpy(b->d_cw64, weights, sizeof(double) * b->n_weights, cudaMemcpyHostToDevice));
  RK_CUDA(cudaMemcpy(b->d_cb64, cb.data(), sizeof(double) * b->K, cudaMemcpyHostToDevice));
  b->f64_ready.store(true, std::memory_order_release);
  return RK_OK;
}

// ---- stateless drop-in for engine._run_batch ----------------------------
namespace {
struct CacheKey {
  const void* p[10];
  int64_t K;
  int C, L;
  uint64_t hash;
  bool operator<(const CacheKey& o) const {
    return std::memcmp(this, &o, sizeof(CacheKey)) < 0;
  }
};
std::mutex g_cache_mu;
// shared ownership: evicting an entry never frees a bank another caller is
// still transforming with (the last reference destroys it)
std::map<CacheKey, std::shared_ptr<rk_bank_s>> g_cache;

uint64_t fnv(uint64_t h, const void* data, size_t bytes) {
  const unsigned char* c = (const unsigned char*)data;
  for (size_t i = 0; i < bytes; ++i) {
    h ^= c[i];
    h *= 1099511628211ull;
  }
  return h;
}
}  // namespace

namespace {
// Shared body of the stateless entry points: look the bank up in the cache
// (identity + content of the arrays), build it on a miss, transform.
int64_t run_batch_impl(int dtype, const void* x, int64_t n_inst, int32_t C, int32_t L, const int32_t* lengths,
                       const int32_t* dilations, const int32_t* paddings, const void* biases, const void* wflat,
                       const int64_t* woff, const int32_t* chidx, const int64_t* choff, const int32_t* chcnt,
                       int64_t K, int32_t workers, int32_t fpk, void* out, int64_t ld_out, int64_t row0,
                       int32_t mode) {
  if (mode != RK_MODE_EXACT && mode != RK_MODE_FAST) return -fail(RK_ERR_INVALID, "unknown mode %d", mode);
  if (workers < 1) return -fail(RK_ERR_INVALID, "workers_per_cell must be positive");
  if (K < 1) return -fail(RK_ERR_INVALID, "bank must contain at least one kernel");
  if (!lengths || !dilations || !paddings || !biases || !wflat || !woff || !chidx || !choff || !chcnt)
    return -fail(RK_ERR_INVALID, "bank array pointer is NULL");
  const int esz = dtype == RK_DTYPE_F64 ? 8 : 4;
  int64_t nw = 0, nci = 0;
  for (int64_t k = 0; k < K; ++k) {
    nw = std::max<int64_t>(nw, woff[k] + (int64_t)lengths[k] * chcnt[k]);
    nci = std::max<int64_t>(nci, choff[k] + chcnt[k]);
  }
  CacheKey key;
  std::memset(&key, 0, sizeof(key));
  const void* ptrs[10] = {lengths, dilations, paddings, biases, wflat, woff, chidx, choff, chcnt, nullptr};
  for (int i = 0; i < 10; ++i) key.p[i] = ptrs[i];
  key.K = K;
  key.C = C;
  key.L = L;
  uint64_t h = 1469598103934665603ull ^ (uint64_t)dtype;
  h = fnv(h, lengths, 4 * K);
  h = fnv(h, dilations, 4 * K);
  h = fnv(h, paddings, 4 * K);
  h = fnv(h, biases, esz * K);
  h = fnv(h, chcnt, 4 * K);
  h = fnv(h, wflat, esz * nw);
  h = fnv(h, chidx, 4 * nci);
  key.hash = h;
  std::shared_ptr<rk_bank_s> bank;
  {
    std::lock_guard<std::mutex> lk(g_cache_mu);
    auto it = g_cache.find(key);
    if (it != g_cache.end()) bank = it->second;
  }
  if (!bank) {
    rk_bank_t created = nullptr;
    int dev = 0;
    cudaGetDevice(&dev);
    std::vector<float> b32, w32;
    const float* bf = static_cast<const float*>(biases);
    const float* wf = static_cast<const float*>(wflat);
    if (esz == 8) {
      const double* bd = static_cast<const double*>(biases);
      const double* wd = static_cast<const double*>(wflat);
      b32.assign(bd, bd + K);
      w32.assign(wd, wd + nw);
      bf = b32.data();
      wf = w32.data();
    }
    int rc = rk_bank_create(K, C, L, lengths, dilations, paddings, bf, wf, woff, chidx, choff, chcnt, dev, &created);
    if (rc) return -rc;
    bank.reset(created, [](rk_bank_s* p) { rk_bank_destroy(p); });
    if (esz == 8) {
      rc = rk_bank_attach_f64(bank.get(), static_cast<const double*>(biases), static_cast<const double*>(wflat));
      if (rc) return -rc;
    }
    std::lock_guard<std::mutex> lk(g_cache_mu);
    if (g_cache.size() >= 8 && !g_cache.count(key)) g_cache.erase(g_cache.begin());
    g_cache[key] = bank;
  }
  int64_t executed = 0;
  int rc = rk_transform(bank.get(), x, dtype, n_inst, out, ld_out, row0, fpk, mode, nullptr, &executed);
  if (rc) return -rc;
  return executed;
}
}  // namespace

int64_t rk_run_batch_f32(const float* x, int64_t n_inst, int32_t C, int32_t L, const int32_t* lengths,
                         const int32_t* dilations, const int32_t* paddings, const float* biases,
                         const float* wflat, const int64_t* woff, const int32_t* chidx, const int64_t* choff,
                         const int32_t* chcnt, int64_t K, int32_t workers, int32_t fpk, float* out,
                         int64_t ld_out, int64_t row0) {
  return run_batch_impl(RK_DTYPE_F32, x, n_inst, C, L, lengths, dilations, paddings, biases, wflat, woff, chidx,
                        choff, chcnt, K, workers, fpk, out, ld_out, row0, RK_MODE_EXACT);
}

int64_t rk_run_batch_f32_mode(const float* x, int64_t n_inst, int32_t C, int32_t L, const int32_t* lengths,
                              const int32_t* dilations, const int32_t* paddings, const float* biases,
                              const float* wflat, const int64_t* woff, const int32_t* chidx, const int64_t* choff,
                              const int32_t* chcnt, int64_t K, int32_t workers, int32_t fpk, float* out,
                              int64_t ld_out, int64_t row0, int32_t mode) {
  return run_batch_impl(RK_DTYPE_F32, x, n_inst, C, L, lengths, dilations, paddings, biases, wflat, woff, chidx,
                        choff, chcnt, K, workers, fpk, out, ld_out, row0, mode);
}

int64_t rk_run_batch_f64(const double* x, int64_t n_inst, int32_t C, int32_t L, const int32_t* lengths,
                         const int32_t* dilations, const int32_t* paddings, const double* biases,
                         const double* wflat, const int64_t* woff, const int32_t* chidx, const int64_t* choff,
                         const int32_t* chcnt, int64_t K, int32_t workers, int32_t fpk, double* out,
                         int64_t ld_out, int64_t row0) {
  return run_batch_impl(RK_DTYPE_F64, x, n_inst, C, L, lengths, dilations, paddings, biases, wflat, woff, chidx,
                        choff, chcnt, K, workers, fpk, out, ld_out, row0, RK_MODE_EXACT);
}

int64_t rk_run_batch_f64_mode(const double* x, int64_t n_inst, int32_t C, int32_t L, const int32_t* lengths,
                              const int32_t* dilations, const int32_t* paddings, const double* biases,
                              const double* wflat, const int64_t* woff, const int32_t* chidx, const int64_t* choff,
                              const int32_t* chcnt, int64_t K, int32_t workers, int32_t fpk, double* out,
                              int64_t ld_out, int64_t row0, int32_t mode) {
  return run_batch_impl(RK_DTYPE_F64, x, n_inst, C, L, lengths, dilations, paddings, biases, wflat, woff, chidx,
                        choff, chcnt, K, workers, fpk, out, ld_out, row0, mode);
}

int rk_release_caches(void) {
  rk_stream_release();
  {
    std::lock_guard<std::mutex> lk(g_cache_mu);
    g_cache.clear();  // banks still in use are destroyed by their last user
  }
  std::lock_guard<std::mutex> lk(g_dev_mu);
  for (auto& kv : g_devs) {
    DeviceState* st = kv.second;
    cudaSetDevice(kv.first);
    std::lock_guard<std::mutex> pl(st->pool_mu);
    for (Worker* w : st->free_workers) {
      for (int i = 0; i < kInBufs; ++i) {
        cudaFree(w->d_in[i]);
        cudaEventDestroy(w->in_ready[i]);
        cudaEventDestroy(w->in_free[i]);
      }
      for (int i = 0; i < kOutBufs; ++i) {
        cudaFree(w->d_out[i]);
        cudaEventDestroy(w->out_ready[i]);
        cudaEventDestroy(w->out_free[i]);
      }
      cudaFree(w->d_scratch);
      cudaStreamDestroy(w->stream);
      cudaStreamDestroy(w->h2d_stream);
      cudaStreamDestroy(w->d2h_stream);
      delete w;
    }
    st->free_workers.clear();
    for (auto& kv : st->gmem_rows) cudaFree(kv.second.p);
    st->gmem_rows.clear();
  }
  return RK_OK;
}

}  // extern "C"
