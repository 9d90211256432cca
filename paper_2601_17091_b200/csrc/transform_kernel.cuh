// transform_kernel.cuh — the sm_100a ROCKET transform kernel.
//
// Replaces the numba hot loop _run_batch (reference:
// /root/reference/pkg/src/gridrocket/engine.py:148-190).  For every
// (series, kernel) cell it evaluates all l_out dot products of the dilated
// kernel and pools them to PPV (positive count / l_out) and MAX, without
// materialising the convolution output.
//
// Work decomposition:
//   * CTA  = one staged series (all channels + zero halos in shared memory)
//            and a block of "chunks" of the device bank;
//   * warp = one chunk: up to 4 kernels (2 FFMA2 pairs) sharing
//            (length, dilation, padding, channel set);
//   * lane = R output positions u, u+d, ..., u+(R-1)d (stride = dilation),
//            so one register window of R+LEN-1 series values feeds
//            R*LEN taps of every kernel in the chunk.
// Kernel pairs are packed into FFMA2 (sm_100 packed FP32) with the series
// value as the scalar-broadcast operand.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace rk {

constexpr int kThreads = 256;      // 8 warps per CTA
constexpr int kMinBlocks = 2;      // 2 CTAs / SM  -> <= 128 registers
constexpr int kChunkKernels = 4;   // kernels per chunk (2 FFMA2 pairs)
constexpr unsigned kFull = 0xffffffffu;

// Class encoding: cls = ((len_idx * kNumR) + r_idx) * 3 + nc_kind
constexpr int kNumR = 4;
__host__ __device__ constexpr int r_of(int r_idx) { return 2 * r_idx + 1; }  // 1,3,5,7
constexpr int kNumClasses = 3 * kNumR * 3;

// One warp work unit.  All kernels of a chunk have the same length,
// dilation, padding and channel set, hence the same valid centre-position
// range [lo, lo + n) (n == l_out, engine.py:163).
struct __align__(16) DevChunk {
  int len;    // taps: 7, 9 or 11
  int d;      // dilation
  int lo;     // first centre position u = t - p + c*d at t = 0
  int n;      // l_out
  int nk;     // live kernel slots (1..4)
  int nc;     // channel slots
  int cls;    // dispatch class
  int wofs;   // float offset into the packed weights
  int chofs;  // offset into the channel-slot table (smem offsets)
  int pad_[3];
  int col[4];     // bank index of each kernel slot
  float thr[4];   // count threshold: exact -> -bias, fast -> 0
  float bias[4];  // exact: added to the max at the end; fast: acc init
};
static_assert(sizeof(DevChunk) == 96, "DevChunk layout");

struct LaunchArgs {
  const float* x;          // (n_series, C, L) device
  float* out;              // row 0 of this launch (already offset by row0)
  int64_t ld_out;          // floats per output row
  int64_t n_items;         // ceil(n_series / series_per_item) * n_blocks (this class)
  int64_t n_series;
  const DevChunk* chunks;  // device, class-sorted
  const float* weights;    // device, packed [slot][pair][tap][2]
  const int* chan_off;     // device, per chunk slot: smem float offset of channel
  const int* block_start;  // device, n_blocks + 1 chunk boundaries (this class)
  unsigned long long* executed;  // device counter
  int n_blocks;
  int series_per_item;     // series staged together (small classes)
  int n_channels;
  int l_series;
  int halo;
  int sstride;             // floats per staged channel (>= L + 2*halo)
  int fpk;
  int vec_out;             // 1 -> 8-byte stores of (ppv, max) are aligned
  int vec_in;              // 1 -> float4 staging loads are aligned
  float one;               // 1.0f, opaque to ptxas (keeps FMUL2 + FFMA2 unfused)
};

__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) { return __ffma2_rn(a, b, c); }
__device__ __forceinline__ float2 fmul2(float2 a, float2 b) { return __fmul2_rn(a, b); }

__device__ __forceinline__ float warp_max(float v) {
  // order-preserving int mapping, then one REDUX.MAX
  int i = __float_as_int(v);
  int key = i >= 0 ? i : (i ^ 0x7fffffff);
  key = __reduce_max_sync(kFull, key);
  int back = key >= 0 ? key : (key ^ 0x7fffffff);
  return __int_as_float(back);
}

// Accumulate one channel slot of a window into acc for P kernel pairs.
// EXACT: acc = RN(acc + RN(w*x)) per tap (FMUL2, then FFMA2 with an opaque
// 1.0 so the product is rounded on its own; reference.py:7-16).
template <int LEN, int R, int P, bool EXACT, bool FIRST>
__device__ __forceinline__ void accumulate(float2 (&acc)[P][R], const float2 (&w)[P][LEN],
                                           const float (&xw)[R + LEN - 1], float2 one2) {
#pragma unroll
  for (int j = 0; j < LEN; ++j) {
#pragma unroll
    for (int p = 0; p < P; ++p) {
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const float2 xv = make_float2(xw[r + j], xw[r + j]);
        if (EXACT) {
          const float2 prod = fmul2(w[p][j], xv);
          if (FIRST && j == 0) acc[p][r] = prod;
          else acc[p][r] = ffma2(prod, one2, acc[p][r]);
        } else {
          acc[p][r] = ffma2(w[p][j], xv, acc[p][r]);
        }
      }
    }
  }
}

template <int LEN, int R, bool MASKED>
__device__ __forceinline__ void load_window(float (&xw)[R + LEN - 1], const float* __restrict__ chan,
                                            int u0, int d, int lo_clamp, int hi_clamp) {
  constexpr int C = (LEN - 1) / 2;
#pragma unroll
  for (int q = 0; q < R + LEN - 1; ++q) {
    int idx = u0 + (q - C) * d;
    if (MASKED) idx = min(max(idx, lo_clamp), hi_clamp);
    xw[q] = chan[idx];
  }
}

// Per-lane pooled state for the kernels of one chunk.
template <int G>
struct Pool {
  unsigned cnt[G];
  float mx[G];
};

template <int LEN, int R, int P, bool EXACT, bool MASKED>
__device__ __forceinline__ void pool_update(Pool<2 * P>& st, const float2 (&acc)[P][R],
                                            const float (&thr)[2 * P], int v0, int d, int n,
                                            bool live) {
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const bool ok = !MASKED || (live && (v0 + r * d < n));
#pragma unroll
    for (int p = 0; p < P; ++p) {
      const float a0 = acc[p][r].x, a1 = acc[p][r].y;
      if (ok) {
        st.cnt[2 * p] += (a0 > thr[2 * p]) ? 1u : 0u;
        st.cnt[2 * p + 1] += (a1 > thr[2 * p + 1]) ? 1u : 0u;
        st.mx[2 * p] = fmaxf(st.mx[2 * p], a0);
        st.mx[2 * p + 1] = fmaxf(st.mx[2 * p + 1], a1);
      }
    }
  }
}

// Finish one chunk: reduce the per-lane pools over the warp and store
// out[row, col*fpk] = ppv, out[row, col*fpk + 1] = max (engine.py:186-188).
template <int G, bool EXACT>
__device__ __forceinline__ void finish_chunk(const DevChunk& c, Pool<G>& st, float* __restrict__ orow,
                                             int fpk, int vec_out, int lane) {
  const double ln = (double)c.n;
#pragma unroll
  for (int g = 0; g < G; ++g) {
    const unsigned tot = __reduce_add_sync(kFull, st.cnt[g]);
    const float m = warp_max(st.mx[g]);
    if (lane == g && g < c.nk) {
      // ppv: count / l_out divided in float64, stored as float32 (engine.py:187)
      const float ppv = __double2float_rn(__ddiv_rn((double)tot, ln));
      const float mx = EXACT ? __fadd_rn(m, c.bias[g]) : m;
      float* dst = orow + (int64_t)c.col[g] * fpk;
      if (vec_out) {
        *reinterpret_cast<float2*>(dst) = make_float2(ppv, mx);
      } else {
        dst[0] = ppv;
        dst[1] = mx;
      }
    }
  }
}

// One chunk with NC channel slots (NC = 1 or 2, weights resident in
// registers) — the fast path for every univariate bank.
template <int LEN, int R, int P, int NC, bool EXACT>
__device__ __forceinline__ void run_chunk(const DevChunk& c, const float* __restrict__ sx,
                                       const float* __restrict__ weights, const int* __restrict__ chan_off,
                                       float* __restrict__ orow, int fpk, int vec_out, int halo, int L,
                                       float one, int lane) {
  constexpr int G = 2 * P;
  constexpr int W = R + LEN - 1;
  float2 w[NC][P][LEN];
  const float2* wp = reinterpret_cast<const float2*>(weights + c.wofs);
#pragma unroll
  for (int s = 0; s < NC; ++s)
#pragma unroll
    for (int p = 0; p < P; ++p)
#pragma unroll
      for (int j = 0; j < LEN; ++j) w[s][p][j] = __ldg(wp + (s * P + p) * LEN + j);
  const float* chan[NC];
#pragma unroll
  for (int s = 0; s < NC; ++s) chan[s] = sx + __ldg(chan_off + c.chofs + s);
  float thr[G];
  float2 init[P];
#pragma unroll
  for (int g = 0; g < G; ++g) thr[g] = EXACT ? c.thr[g] : 0.0f;
#pragma unroll
  for (int p = 0; p < P; ++p) init[p] = make_float2(c.bias[2 * p], c.bias[2 * p + 1]);
  Pool<G> st;
#pragma unroll
  for (int g = 0; g < G; ++g) {
    st.cnt[g] = 0u;
    st.mx[g] = -INFINITY;
  }
  const float2 one2 = make_float2(one, one);
  const int d = c.d, n = c.n, lo = c.lo;
  const int RD = R * d;
  const int A = n / RD;
  const int rem = n - A * RD;
  const int starts = A * d + min(d, rem);
  const int lo_clamp = -halo, hi_clamp = L + halo - 1;
  for (int base = 0; base < starts; base += 32) {
    const int i = base + lane;
    const bool live = i < starts;
    const int ii = live ? i : 0;
    const int a = ii / d;
    const int s0 = ii - a * d;
    const int v0 = a * RD + s0;
    const int u0 = lo + v0;
    const bool full = __all_sync(kFull, live && (v0 + (R - 1) * d < n));
    float2 acc[P][R];
    if (full) {
#pragma unroll
      for (int s = 0; s < NC; ++s) {
        float xw[W];
        load_window<LEN, R, false>(xw, chan[s], u0, d, lo_clamp, hi_clamp);
        if (s == 0) {
          if (!EXACT) {
#pragma unroll
            for (int p = 0; p < P; ++p)
#pragma unroll
              for (int r = 0; r < R; ++r) acc[p][r] = init[p];
            accumulate<LEN, R, P, EXACT, false>(acc, w[s], xw, one2);
          } else {
            accumulate<LEN, R, P, EXACT, true>(acc, w[s], xw, one2);
          }
        } else {
          accumulate<LEN, R, P, EXACT, false>(acc, w[s], xw, one2);
        }
      }
      pool_update<LEN, R, P, EXACT, false>(st, acc, thr, v0, d, n, live);
    } else {
#pragma unroll
      for (int s = 0; s < NC; ++s) {
        float xw[W];
        load_window<LEN, R, true>(xw, chan[s], u0, d, lo_clamp, hi_clamp);
        if (s == 0) {
          if (!EXACT) {
#pragma unroll
            for (int p = 0; p < P; ++p)
#pragma unroll
              for (int r = 0; r < R; ++r) acc[p][r] = init[p];
            accumulate<LEN, R, P, EXACT, false>(acc, w[s], xw, one2);
          } else {
            accumulate<LEN, R, P, EXACT, true>(acc, w[s], xw, one2);
          }
        } else {
          accumulate<LEN, R, P, EXACT, false>(acc, w[s], xw, one2);
        }
      }
      pool_update<LEN, R, P, EXACT, true>(st, acc, thr, v0, d, n, live);
    }
  }
  finish_chunk<G, EXACT>(c, st, orow, fpk, vec_out, lane);
}

// Generic channel count (>= 3 slots): one kernel pair, weights re-read
// from L1 per slot and step.
template <int LEN, int R, bool EXACT>
__device__ __forceinline__ void run_chunk_generic(const DevChunk& c, const float* __restrict__ sx,
                                               const float* __restrict__ weights,
                                               const int* __restrict__ chan_off, float* __restrict__ orow,
                                               int fpk, int vec_out, int halo, int L, float one, int lane) {
  constexpr int P = 1;
  constexpr int G = 2;
  constexpr int W = R + LEN - 1;
  const float2* wp = reinterpret_cast<const float2*>(weights + c.wofs);
  float thr[G] = {EXACT ? c.thr[0] : 0.0f, EXACT ? c.thr[1] : 0.0f};
  const float2 init = make_float2(c.bias[0], c.bias[1]);
  Pool<G> st;
#pragma unroll
  for (int g = 0; g < G; ++g) {
    st.cnt[g] = 0u;
    st.mx[g] = -INFINITY;
  }
  const float2 one2 = make_float2(one, one);
  const int d = c.d, n = c.n, lo = c.lo, nc = c.nc;
  const int RD = R * d;
  const int A = n / RD;
  const int rem = n - A * RD;
  const int starts = A * d + min(d, rem);
  const int lo_clamp = -halo, hi_clamp = L + halo - 1;
  for (int base = 0; base < starts; base += 32) {
    const int i = base + lane;
    const bool live = i < starts;
    const int ii = live ? i : 0;
    const int a = ii / d;
    const int s0 = ii - a * d;
    const int v0 = a * RD + s0;
    const int u0 = lo + v0;
    float2 acc[P][R];
    for (int s = 0; s < nc; ++s) {
      float2 w[P][LEN];
#pragma unroll
      for (int j = 0; j < LEN; ++j) w[0][j] = __ldg(wp + s * LEN + j);
      float xw[W];
      load_window<LEN, R, true>(xw, sx + __ldg(chan_off + c.chofs + s), u0, d, lo_clamp, hi_clamp);
      if (s == 0) {
        if (!EXACT) {
#pragma unroll
          for (int r = 0; r < R; ++r) acc[0][r] = init;
          accumulate<LEN, R, P, EXACT, false>(acc, w, xw, one2);
        } else {
          accumulate<LEN, R, P, EXACT, true>(acc, w, xw, one2);
        }
      } else {
        accumulate<LEN, R, P, EXACT, false>(acc, w, xw, one2);
      }
    }
    pool_update<LEN, R, P, EXACT, true>(st, acc, thr, v0, d, n, live);
  }
  finish_chunk<G, EXACT>(c, st, orow, fpk, vec_out, lane);
}

// One launch per chunk class <LEN, R, NCK>: each class gets its own
// register allocation and straight-line code (no dispatch in the warp loop).
// Items are (series, block of this class's chunks); a CTA stages the series
// once per item and its warps pull chunks with a shared-memory counter.
template <int LEN, int R, int NCK, bool EXACT>
__global__ void __launch_bounds__(kThreads, kMinBlocks) rocket_class_kernel(const LaunchArgs a) {
  extern __shared__ __align__(16) float smem[];
  __shared__ int s_next;
  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int C = a.n_channels, L = a.l_series, H = a.halo, S = a.sstride;
  const int SPI = a.series_per_item;
  const int slot_floats = C * S;
  // Zero the halos once; only the interiors are rewritten per series.
  for (int k = tid; k < SPI * slot_floats; k += kThreads) {
    const int t = (k % slot_floats) % S;
    if (t < H || t >= H + L) smem[k] = 0.0f;
  }
  unsigned long long done = 0;
  for (int64_t item = blockIdx.x; item < a.n_items; item += gridDim.x) {
    const int64_t group = item / a.n_blocks;
    const int blk = (int)(item - group * a.n_blocks);
    const int64_t series0 = group * SPI;
    const int64_t left = a.n_series - series0;
    const int ns = left < SPI ? (int)left : SPI;
    __syncthreads();  // every warp has left the previous item
    const float* xs = a.x + series0 * (int64_t)C * L;
    if (a.vec_in) {
      const int L4 = L >> 2;
      for (int k = tid; k < ns * C * L4; k += kThreads) {
        const int row = k / L4, t = k - row * L4;  // row = series * C + channel
        const float4 v = __ldg(reinterpret_cast<const float4*>(xs + (int64_t)row * L) + t);
        float* dst = smem + row * S + H + 4 * t;
        dst[0] = v.x; dst[1] = v.y; dst[2] = v.z; dst[3] = v.w;
      }
    } else {
      for (int k = tid; k < ns * C * L; k += kThreads) {
        const int row = k / L, t = k - row * L;
        smem[row * S + H + t] = __ldg(xs + k);
      }
    }
    if (tid == 0) s_next = 0;
    __syncthreads();
    const int cbeg = __ldg(a.block_start + blk);
    const int nchunk = __ldg(a.block_start + blk + 1) - cbeg;
    const int nwork = nchunk * ns;
    while (true) {
      int w = 0;
      if (lane == 0) w = atomicAdd(&s_next, 1);
      w = __shfl_sync(kFull, w, 0);
      if (w >= nwork) break;
      const int ci = cbeg + w / ns;  // chunk-major: consecutive warps share weights in L1
      const int si = w - (w / ns) * ns;
      const DevChunk c = a.chunks[ci];
      float* orow = a.out + (series0 + si) * a.ld_out;
      const float* sx = smem + si * slot_floats + H;  // chan_off entries are relative to this
      if (NCK == 0)
        run_chunk<LEN, R, 2, 1, EXACT>(c, sx, a.weights, a.chan_off, orow, a.fpk, a.vec_out, H, L, a.one, lane);
      else if (NCK == 1)
        run_chunk<LEN, R, 1, 2, EXACT>(c, sx, a.weights, a.chan_off, orow, a.fpk, a.vec_out, H, L, a.one, lane);
      else
        run_chunk_generic<LEN, R, EXACT>(c, sx, a.weights, a.chan_off, orow, a.fpk, a.vec_out, H, L, a.one, lane);
      done += (unsigned long long)c.nk * (unsigned long long)c.n;
    }
  }
  if (lane == 0 && done) atomicAdd(a.executed, done);
}

}  // namespace rk
