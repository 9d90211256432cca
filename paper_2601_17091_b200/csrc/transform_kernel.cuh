// transform_kernel.cuh — the sm_100a ROCKET transform kernels.
//
// Replaces the numba hot loop _run_batch (reference:
// /root/reference/pkg/src/gridrocket/engine.py:148-190).  For every
// (series, kernel) cell it evaluates all l_out dot products of the dilated
// kernel and pools them to PPV (positive count / l_out) and MAX, without
// materialising the convolution output.
//
// Work decomposition:
//   * chunk = up to 4 kernels (2 FFMA2 pairs) sharing (dilation, centre
//             range [lo, lo+n), channel set) — one warp work unit;
//   * lane  = R output positions u, u+d, ..., u+(R-1)d (stride = dilation),
//             so one register window of R+LEN-1 series values feeds
//             R*LEN taps of every kernel of the chunk;
//   * kernel pairs are packed into FFMA2 (sm_100 packed FP32) with the
//     series value as the scalar-broadcast operand.
// Two kernels drive it:
//   * rocket_wide_kernel  (chunks with <= 2 channel slots): chunk
//     descriptors and weights travel in the __grid_constant__ parameter
//     block, so the weights sit in uniform registers (FFMA2 UR operands);
//     W warps per CTA share one staged series;
//   * rocket_class_kernel (banks with >= 3-channel kernels): 16-warp CTAs
//     share one staged series, weights come from global memory.
//
// Arithmetic (both modes are deterministic run to run):
//   EXACT: acc = RN(acc + RN(w*x)) tap by tap from the first product
//          (FMUL2, then FFMA2 with an opaque 1.0 so ptxas cannot contract
//          the pair), channels then taps ascending, zero halos add +-0
//          (never changes the sum).  Pooling compares acc > -bias
//          (RN(acc + b) > 0 <=> acc > -b exactly) and the max is
//          RN(max_t acc_t + b) == max_t RN(acc_t + b) — bit-identical to
//          the reference (reference.py:1-17, engine.py:172-188).
//   FAST:  the series is staged negated and the accumulator starts at -b,
//          so acc' = -(b + sum w*x) via FFMA2 only.  "output > 0" is then
//          the sign bit of acc' (acc' is never -0: its init is never -0
//          and RN sums of non-(-0) terms are +0 when exactly zero), counted
//          with one shift-add, and MAX = -min(acc').
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace rk {

#ifndef RK_THREADS
#define RK_THREADS 512
#endif
#ifndef RK_MINBLOCKS
#define RK_MINBLOCKS 1
#endif
#ifndef RK_RMAX
#define RK_RMAX 11
#endif
#ifndef RK_UNROLL
#define RK_UNROLL 2
#endif
constexpr int kStepUnroll = RK_UNROLL;    // full-step loop unroll
constexpr int kThreads = RK_THREADS;      // class kernel: 16 warps per CTA
constexpr int kMinBlocks = RK_MINBLOCKS;  // class kernel: 1 CTA / SM (<= 128 registers)
constexpr unsigned kFull = 0xffffffffu;

// Class encoding: cls = ((len_idx * kNumR) + r_idx) * kNumNck + nc_kind
//   nc_kind 0: 1 channel, 2 kernel pairs; 1: 2 channels, 1 pair;
//           2: >= 3 channels, 1 pair (wide kernel: channel slots looped at
//              run time; class kernel: the generic 1-position path);
//           3: 1 channel, 1 pair; 4 / 5: kinds 0 / 3 as half-warp chunks;
//           6 / 7: one kernel over 1 / 2 channels, position-paired
#ifndef RK_NUM_R
#define RK_NUM_R 8
#endif
constexpr int kNumR = RK_NUM_R;  // R = 1, 3, 5, 7, RK_RMAX (11), 13, 9, 15
// positions per lane of class r_idx: 1, 3, 5, 7, RK_RMAX, 13, 9, 15 (odd:
// spreads lanes over the shared-memory banks); the cost model picks one per
// chunk.
__host__ __device__ constexpr int r_of(int r_idx) {
  return r_idx == 7 ? 15 : r_idx == 6 ? 9 : r_idx == 5 ? 13 : r_idx == 4 ? RK_RMAX : 2 * r_idx + 1;
}
// exact mode and fast-mode MPV: R <= 13 (their FMUL2 temporaries / partial
// sums spill at 15); a larger class runs at the R = 13 index
constexpr int kExactRMax = 13;
constexpr int kExactRIdx13 = 5;
static_assert(r_of(kExactRIdx13) == kExactRMax, "R class table");
constexpr int kNumNck = 12;
// (P, NC) of a channel kind on the wide path; NC = 0: run-time slot loop.
// 4 / 5: the 1-channel kinds 0 / 3 run as half-warp chunks (two series per
// pass); same chunk data, so they fall back to 0 / 3 when items hold one
// series.  6 / 7: single-kernel chunks over 1 / 2 channel slots run
// position-paired ("SP"): the two FFMA2 lanes hold two positions of the
// one kernel instead of a kernel and an idle zero-weight slot.
// 8 / 9: the 1-channel kinds 0 / 3 as quarter-warp chunks (four series per
// pass, 8 lanes each); 10 / 11: as eighth-warp chunks (eight series per
// pass, 4 lanes each).  A transform whose items hold fewer series than a
// kind's groups runs a narrower twin layout of the bank.
__host__ __device__ constexpr int nck_pairs(int nck) { return (nck == 0 || nck == 4 || nck == 8 || nck == 10) ? 2 : 1; }
__host__ __device__ constexpr int nck_slots(int nck) { return (nck == 1 || nck == 7) ? 2 : nck == 2 ? 0 : 1; }
__host__ __device__ constexpr bool nck_half(int nck) { return nck == 4 || nck == 5; }
__host__ __device__ constexpr bool nck_quarter(int nck) { return nck == 8 || nck == 9; }
__host__ __device__ constexpr bool nck_eighth(int nck) { return nck == 10 || nck == 11; }
__host__ __device__ constexpr bool nck_sp(int nck) { return nck == 6 || nck == 7; }
// lanes per series group of a kind (32: the whole warp on one series)
__host__ __device__ constexpr int nck_lanes(int nck) {
  return nck_half(nck) ? 16 : nck_quarter(nck) ? 8 : nck_eighth(nck) ? 4 : 32;
}
// series per pass of a kind (1, 2, 4, 8)
__host__ __device__ constexpr int nck_groups(int nck) { return 32 / nck_lanes(nck); }
// largest R of the position-paired kinds (2R positions per lane: the pair
// window and accumulators fit the ~80-register budget; one slot walks its
// window anti-diagonally, see chunk_step_sp)
__host__ __device__ constexpr int sp_rmax(int nc, int len) { return nc == 1 ? 15 : 5; }
__host__ __device__ constexpr int nck_full(int nck) {
  return (nck == 4 || nck == 8 || nck == 10) ? 0 : (nck == 5 || nck == 9 || nck == 11) ? 3 : nck;
}
constexpr int kNumClasses = 3 * kNumR * kNumNck;

// One chunk (class-kernel layout, global memory).
struct __align__(16) DevChunk {
  int len;    // taps: 7, 9 or 11 (shorter kernels zero-padded inside)
  int d;      // dilation
  int lo;     // first centre position u = t - p + c*d at t = 0
  int n;      // l_out
  int nk;     // live kernel slots (1..4)
  int nc;     // channel slots
  int cls;    // dispatch class
  int wofs;   // float offset into the packed weights
  int chofs;  // offset into the channel-slot table (smem offsets)
  int q32;    // 32 / d       (lane map, precomputed on the host)
  int r32;    // 32 % d
  float invd; // 1 / d        (lane / d for lane < 32 via one multiply)
  int col[4];     // bank index of each kernel slot
  float thr[4];   // exact: count threshold -bias (+0.0f, never -0)
  float bias[4];  // bias (+0.0f: never -0)
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
  int* item_counter;       // dynamic item scheduler (zeroed before the launch)
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

// ---- checked build (-DRK_CHECKED): device-side bounds checks ------------
// compute-sanitizer is closed on the GPU pool, so the library carries its
// own memory checks: every window read must fall inside the CTA's dynamic
// shared memory (or the canonical NaN slot), or — for series read from
// global memory — inside the zero-haloed row scratch; every feature store
// inside rows [0, n_series) of the launch's output; __trap() otherwise.
// Without RK_CHECKED the macros are empty and the kernels are unchanged.
#ifdef RK_CHECKED
__shared__ unsigned rk_chk_s_lo, rk_chk_s_hi;          // dynamic smem [lo, hi)
__shared__ const void* rk_chk_nan;                     // the canonical NaN slot
__shared__ const char *rk_chk_g_lo, *rk_chk_g_hi;      // global series rows
__shared__ const char *rk_chk_o_lo, *rk_chk_o_hi;      // output rows
__device__ __forceinline__ unsigned rk_dyn_smem_bytes() {
  unsigned v;
  asm volatile("mov.u32 %0, %%dynamic_smem_size;" : "=r"(v));
  return v;
}
__device__ __forceinline__ void rk_chk_set(const void* smem_base, const void* nan, const void* g_lo,
                                           const void* g_hi, const void* o_lo, const void* o_hi) {
  rk_chk_s_lo = static_cast<unsigned>(__cvta_generic_to_shared(smem_base));
  rk_chk_s_hi = rk_chk_s_lo + rk_dyn_smem_bytes();
  rk_chk_nan = nan;
  rk_chk_g_lo = static_cast<const char*>(g_lo);
  rk_chk_g_hi = static_cast<const char*>(g_hi);
  rk_chk_o_lo = static_cast<const char*>(o_lo);
  rk_chk_o_hi = static_cast<const char*>(o_hi);
}
__device__ __forceinline__ void rk_chk_read(const void* a, int bytes) {
  if (a == rk_chk_nan) return;
  if (__isShared(a)) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(a));
    if (s < rk_chk_s_lo || s + bytes > rk_chk_s_hi) __trap();
  } else {
    const char* c = static_cast<const char*>(a);
    if (c < rk_chk_g_lo || c + bytes > rk_chk_g_hi) __trap();
  }
}
__device__ __forceinline__ void rk_chk_write(const void* a, int bytes) {
  const char* c = static_cast<const char*>(a);
  if (c < rk_chk_o_lo || c + bytes > rk_chk_o_hi) __trap();
}
#define RK_CHK_READ(a, bytes) ::rk::rk_chk_read((a), (bytes))
#define RK_CHK_WRITE(a, bytes) ::rk::rk_chk_write((a), (bytes))
#define RK_CHK_SET(...) ::rk::rk_chk_set(__VA_ARGS__)
#define RK_CHK(cond) \
  do {               \
    if (!(cond)) __trap(); \
  } while (0)
#else
#define RK_CHK_READ(a, bytes) ((void)0)
#define RK_CHK_WRITE(a, bytes) ((void)0)
#define RK_CHK_SET(...) ((void)0)
#define RK_CHK(cond) ((void)0)
#endif

__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) { return __ffma2_rn(a, b, c); }
__device__ __forceinline__ float2 fmul2(float2 a, float2 b) { return __fmul2_rn(a, b); }

// order-preserving int key of a float (no NaNs here), for REDUX min/max
__device__ __forceinline__ int fkey(float v) {
  const int i = __float_as_int(v);
  return i >= 0 ? i : (i ^ 0x7fffffff);
}
__device__ __forceinline__ float fkey_inv(int k) { return __int_as_float(k >= 0 ? k : (k ^ 0x7fffffff)); }
__device__ __forceinline__ float warp_max(float v) { return fkey_inv(__reduce_max_sync(kFull, fkey(v))); }
__device__ __forceinline__ float warp_min(float v) { return fkey_inv(__reduce_min_sync(kFull, fkey(v))); }

// Accumulate one channel slot of a window into acc for P kernel pairs.
// FIRST && j == 0 starts the accumulator: EXACT from the first product,
// FAST from init (-bias pair) with the first FFMA2.
template <int LEN, int R, int P, bool EXACT, bool FIRST>
__device__ __forceinline__ void accumulate(float2 (&acc)[P][R], const float2 (&w)[P][LEN],
                                           const float (&xw)[R + LEN - 1], const float2 (&init)[P][R],
                                           float2 one2) {
#pragma unroll
  for (int j = 0; j < LEN; ++j) {
#pragma unroll
    for (int p = 0; p < P; ++p) {
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const float2 xv = make_float2(xw[r + j], xw[r + j]);
        if (EXACT) {
          if (FIRST && j == 0)
            acc[p][r] = fmul2(w[p][j], xv);  // RN(w*x) == RN(+0 + RN(w*x))
          else
            acc[p][r] = ffma2(fmul2(w[p][j], xv), one2, acc[p][r]);
        } else {
          acc[p][r] = ffma2(w[p][j], xv, (FIRST && j == 0) ? init[p][r] : acc[p][r]);
        }
      }
    }
  }
}

template <int LEN, int R>
__device__ __forceinline__ void load_window(float (&xw)[R + LEN - 1], const float* __restrict__ chan, int u0,
                                            int d) {
  constexpr int C = (LEN - 1) / 2;
  const float* p = chan + (u0 - C * d);
#pragma unroll
  for (int q = 0; q < R + LEN - 1; ++q) {
    RK_CHK_READ(p + q * d, 4);
    xw[q] = p[q * d];
  }
}

// Masked steps: a lane's valid positions are a prefix r < rcount of its
// run (rcount = 0 for a lane without a run).  Position r reads window
// entries r .. r+LEN-1, so entry q = r+LEN-1 (its last tap) is loaded only
// while r*d < nleft and otherwise replaced by a canonical NaN: every output
// of a dead position is NaN, which the pooling ignores by IEEE semantics
// (NaN > t is false; min/max return the other operand; the sign bit of the
// canonical NaN is clear, so the FAST count adds nothing).  The first LEN-1
// entries belong to position 0, which is in range for a live lane and is
// read at lane start lo for a dead one.
template <int LEN, int R>
__device__ __forceinline__ void load_window_masked(float (&xw)[R + LEN - 1], const float* __restrict__ chan,
                                                   int u0, int d, int nleft, const float* nan_slot) {
  constexpr int C = (LEN - 1) / 2;
  const float* p = chan + (u0 - C * d);
#pragma unroll
  for (int q = 0; q < R + LEN - 1; ++q) {
    const float* a = p + q * d;
    if (q >= LEN - 1) a = (q - (LEN - 1)) * d < nleft ? a : nan_slot;
    RK_CHK_READ(a, 4);
    xw[q] = *a;
  }
}

// Per-lane pooled state for the kernels of one chunk.  ext is the running
// max (EXACT) or the running min of acc' = -(output) (FAST).
// MPV (FAST only) adds per-pair partial sums of min(acc', 0) = -(positive
// outputs).
template <int G, bool MPV = false>
struct Pool {
  unsigned cnt[G];
  float ext[G];
  float2 ps[MPV ? G / 2 : 1];
};

template <int G, bool EXACT, bool MPV = false>
__device__ __forceinline__ void pool_init(Pool<G, MPV>& st) {
#pragma unroll
  for (int g = 0; g < G; ++g) {
    st.cnt[g] = 0u;
    st.ext[g] = EXACT ? -INFINITY : INFINITY;
  }
  if (MPV) {
#pragma unroll
    for (int q = 0; q < G / 2; ++q) st.ps[q] = make_float2(0.0f, 0.0f);
  }
}

// count += (a > t): FSETP + predicated add, both on the ALU pipe.
__device__ __forceinline__ void count_gt(unsigned& cnt, float a, float t, bool live) {
  asm("{\n\t.reg .pred p, q;\n\tsetp.ne.u32 q, %3, 0;\n\tsetp.gt.and.f32 p, %1, %2, q;\n\t@p add.u32 %0, %0, 1;\n\t}"
      : "+r"(cnt)
      : "f"(a), "f"(t), "r"((unsigned)live));
}

// Pool one output of kernel slot g.
template <bool EXACT, bool MASKED>
__device__ __forceinline__ void pool_one(unsigned& cnt, float& ext, float a, float thr, bool ok) {
  if (EXACT) {
    if (MASKED) {
      count_gt(cnt, a, thr, ok);
      ext = ok ? fmaxf(ext, a) : ext;
    } else {
      count_gt(cnt, a, thr, true);
      ext = fmaxf(ext, a);
    }
  } else {
    // acc' < 0 <=> output > 0; acc' is never -0, so the sign bit decides
    if (MASKED) {
      if (ok) cnt += __float_as_uint(a) >> 31;
      ext = ok ? fminf(ext, a) : ext;
    } else {
      cnt += __float_as_uint(a) >> 31;
      ext = fminf(ext, a);
    }
  }
}

// Pool R positions of P kernel pairs; position r is valid while
// r*d < nleft (MASKED only).
template <int R, int P, bool EXACT, bool MASKED, bool MPV = false>
__device__ __forceinline__ void pool_update(Pool<2 * P, MPV>& st, const float2 (&acc)[P][R],
                                            const float (&thr)[2 * P], bool live, int nleft, int d) {
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const bool ok = !MASKED || (live && (r * d < nleft));
#pragma unroll
    for (int p = 0; p < P; ++p) {
      pool_one<EXACT, MASKED>(st.cnt[2 * p], st.ext[2 * p], acc[p][r].x, thr[2 * p], ok);
      pool_one<EXACT, MASKED>(st.cnt[2 * p + 1], st.ext[2 * p + 1], acc[p][r].y, thr[2 * p + 1], ok);
      if (MPV) {
        // min(NaN, 0) = 0: dead positions of masked steps add nothing
        st.ps[p] = __fadd2_rn(st.ps[p], make_float2(fminf(acc[p][r].x, 0.0f), fminf(acc[p][r].y, 0.0f)));
      }
    }
  }
}

// Finish one chunk: reduce the per-lane pools over the warp; lane g
// finishes kernel g: out[row, col*fpk] = ppv, out[row, col*fpk+1] = max
// (engine.py:186-188).
template <int G, bool EXACT, class CH, bool MPV = false>
__device__ __forceinline__ void finish_chunk(const CH& c, Pool<G, MPV>& st, float* __restrict__ orow, int fpk,
                                             int vec_out, int lane) {
  unsigned my_cnt = 0;
  float my_ext = 0.0f, my_bias = 0.0f, my_ps = 0.0f;
  int my_col = 0;
#pragma unroll
  for (int g = 0; g < G; ++g) {
    const unsigned tot = __reduce_add_sync(kFull, st.cnt[g]);
    const float e = EXACT ? warp_max(st.ext[g]) : warp_min(st.ext[g]);
    float ps = 0.0f;
    if (MPV) {
      ps = (g & 1) ? st.ps[g / 2].y : st.ps[g / 2].x;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) ps += __shfl_xor_sync(kFull, ps, o);
    }
    if (lane == g) {
      my_cnt = tot;
      my_ext = e;
      my_bias = c.bias[g];
      my_col = c.col[g];
      my_ps = ps;
    }
  }
  if (lane < c.nk) {
    // ppv: the reference stores f32(RN64(count / l_out)) (engine.py:187).
    // For integers c <= n < 2^24 that equals the single rounding
    // RN32(c / n): a non-midpoint quotient lies >= 2^-49 (relative) from
    // every f32 midpoint, farther than RN64 moves it, so both roundings pick
    // the same float (checked exhaustively for n <= 20000 and sampled to
    // 2^24, tests/test_host.py).
    const float ppv = __fdiv_rn((float)my_cnt, (float)c.n);
    // exact: RN(max_t acc_t + b) == max_t RN(acc_t + b); fast: -min acc'
    const float mx = EXACT ? __fadd_rn(my_ext, my_bias) : -my_ext;
    float* dst = orow + (int64_t)my_col * fpk;
    RK_CHK_WRITE(dst, (MPV ? 3 : 2) * 4);
    if (vec_out) {
      *reinterpret_cast<float2*>(dst) = make_float2(ppv, mx);
    } else {
      dst[0] = ppv;
      dst[1] = mx;
    }
    // mpv = (sum of positive outputs) / count, divided in float64 like
    // the reference (engine.py:244-247); 0 without positives
    if (MPV) dst[2] = my_cnt ? __double2float_rn((double)(-my_ps) / (double)my_cnt) : 0.0f;
  }
}

// Finish for lane-group chunks (LG = 16: half-warp, 8: quarter-warp):
// lanes [g*LG, (g+1)*LG) hold series si + g's pools; butterfly reductions
// inside each group, then lane k of each group writes kernel k of its
// series (orow: the group's output row, null for a group shadowing the
// last series, which writes nothing).
template <int G, bool EXACT, class CH, bool MPV = false, int LG = 16>
__device__ __forceinline__ void finish_chunk_group(const CH& c, Pool<G, MPV>& st, float* __restrict__ orow, int fpk,
                                                   int vec_out, int lane) {
  const int hl = lane & (LG - 1);
  unsigned my_cnt = 0;
  float my_ext = 0.0f, my_bias = 0.0f, my_ps = 0.0f;
  int my_col = 0;
#pragma unroll
  for (int g = 0; g < G; ++g) {
    unsigned cnt = st.cnt[g];
    float e = st.ext[g];
    float ps = 0.0f;
    if (MPV) ps = (g & 1) ? st.ps[g / 2].y : st.ps[g / 2].x;
#pragma unroll
    for (int o = LG / 2; o > 0; o >>= 1) {
      cnt += __shfl_xor_sync(kFull, cnt, o);
      const float oe = __shfl_xor_sync(kFull, e, o);
      e = EXACT ? fmaxf(e, oe) : fminf(e, oe);
      if (MPV) ps += __shfl_xor_sync(kFull, ps, o);
    }
    if (hl == g) {
      my_cnt = cnt;
      my_ext = e;
      my_bias = c.bias[g];
      my_col = c.col[g];
      my_ps = ps;
    }
  }
  if (hl < c.nk && orow) {
    const float ppv = __fdiv_rn((float)my_cnt, (float)c.n);  // == f32(RN64(count / l_out)), see finish_chunk
    const float mx = EXACT ? __fadd_rn(my_ext, my_bias) : -my_ext;
    float* dst = orow + (int64_t)my_col * fpk;
    RK_CHK_WRITE(dst, (MPV ? 3 : 2) * 4);
    if (vec_out) {
      *reinterpret_cast<float2*>(dst) = make_float2(ppv, mx);
    } else {
      dst[0] = ppv;
      dst[1] = mx;
    }
    if (MPV) dst[2] = my_cnt ? __double2float_rn((double)(-my_ps) / (double)my_cnt) : 0.0f;  // see finish_chunk
  }
}

// One step: R positions per lane (u0, u0+d, ..., u0+(R-1)d) for P kernel
// pairs over NC channel slots.
template <int LEN, int R, int P, int NC, bool EXACT, bool MASKED, bool MPV = false>
__device__ __forceinline__ void chunk_step(Pool<2 * P, MPV>& st, const float* const (&chan)[NC],
                                           const float2 (&w)[NC][P][LEN], const float (&thr)[2 * P],
                                           const float2 (&init)[P], float2 one2, int u0, int d, int nleft,
                                           const float* nan_slot) {
  float2 init_r[P][R];
#pragma unroll
  for (int p = 0; p < P; ++p)
#pragma unroll
    for (int r = 0; r < R; ++r) init_r[p][r] = init[p];
  float2 acc[P][R];
#pragma unroll
  for (int s = 0; s < NC; ++s) {
    float xw[R + LEN - 1];
    if (MASKED)
      load_window_masked<LEN, R>(xw, chan[s], u0, d, nleft, nan_slot);
    else
      load_window<LEN, R>(xw, chan[s], u0, d);
    if (s == 0)
      accumulate<LEN, R, P, EXACT, true>(acc, w[s], xw, init_r, one2);
    else
      accumulate<LEN, R, P, EXACT, false>(acc, w[s], xw, init_r, one2);
  }
  pool_update<R, P, EXACT, false, MPV>(st, acc, thr, true, 0, d);
}

// Lane map.  Positions v in [0, n) (centre u = lo + v) are split into runs
// v = (a*R + r)*d + s, r < R, s < d; run starts i = a*d + s are dealt to
// lanes in consecutive order (consecutive s -> consecutive smem addresses;
// R odd spreads consecutive a over the banks).  Steps whose 32 starts are
// all complete runs go through the unmasked path; the remaining starts
// (an incomplete 32-group and the final partial run, whose positions
// v0 + r*d may pass n) through masked steps with clamped reads.
// LANES = 16 / 8: a half / quarter warp walks one series (lane is the lane
// in its group, q32 / r32 are LANES / d and LANES % d).
//
// Run-major map (amap = log2 g >= 0, chosen per chunk by the host where it
// replays fewer shared-memory wavefronts): the complete-run starts are dealt
// as i -> (sb, a, sl) with sl = i mod g fastest, then the run index a < A,
// then the residue block sb (start s = sb*g + sl), g = the largest power of
// two dividing d (<= LANES).  The LANES starts of a step are then LANES/g
// consecutive runs of g residues: banks a*(R*d) + sl, distinct because R*d/g
// is odd — where the residue-major map above puts d-position blocks R*d
// apart and replays up to 5-way at d = 3, 5, 7, ... .  Both maps are a
// mixed-radix counter (radix d / radix A) advanced by LANES per step.
template <int LEN, int R, int P, int NC, bool EXACT, bool MPV = false, int LANES = 32>
__device__ __forceinline__ void run_positions(Pool<2 * P, MPV>& st, const float* const (&chan)[NC],
                                              const float2 (&w)[NC][P][LEN], const float (&thr)[2 * P],
                                              const float2 (&init)[P], float2 one2, int lo, int n, int d, int q32,
                                              int r32, float invd, const float* nan_slot, int lane,
                                              bool tail = false, int amap = -1) {
  constexpr int kLog = LANES == 32 ? 5 : LANES == 16 ? 4 : LANES == 8 ? 3 : 2;
  const int RD = R * d;
  const int A = n / RD;          // complete runs per residue
  const int rem = n - A * RD;    // positions of the partial run
  const int full_starts = A * d;
  // tail mode: stop at the last complete run; the rem positions [A*R*d, n)
  // — a contiguous range — run below as an R = 1 map
  const int starts = (R > 1 && tail) ? full_starts : full_starts + min(d, rem);
  const int nfull = full_starts >> kLog;
  int t, v0, radix, tstep, vstep, vwrap;
  if (R > 1 && amap >= 0 && A > 0) {
    const int kg = min(amap, kLog), g = 1 << kg;
    const int J = LANES >> kg, qa = J / A, ra = J - qa * A;  // runs per step = qa*A + ra
    const int j = lane >> kg;
    const int sb = j / A;
    t = j - sb * A;  // run index a
    v0 = t * RD + sb * g + (lane & (g - 1));
    radix = A;
    tstep = ra;
    vstep = ra * RD + qa * g;
    vwrap = g - A * RD;
  } else {
    // (a, s) = divmod(32*step + lane, d), advanced incrementally; the first
    // divmod of lane < 32 is exact in float ((lane + 0.5) / d is never within
    // 2^-20 of an integer)
    const int a = (int)((lane + 0.5f) * invd);
    t = lane - a * d;  // residue s
    v0 = a * RD + t;
    radix = d;
    tstep = r32;
    vstep = q32 * RD + r32;
    vwrap = RD - d;
  }
#pragma unroll(kStepUnroll)
  for (int stp = 0; stp < nfull; ++stp) {
    chunk_step<LEN, R, P, NC, EXACT, false, MPV>(st, chan, w, thr, init, one2, lo + v0, d, n, nan_slot);
    t += tstep;
    v0 += vstep;
    if (t >= radix) {
      t -= radix;
      v0 += vwrap;
    }
  }
  for (int base = nfull << kLog; base < starts; base += LANES) {
    // starts past the complete runs (the partial run of each residue) sit at
    // A*R*d + s in both maps
    const int i = base + lane;
    const bool live = i < starts;
    const int v = i < full_starts ? v0 : A * RD + (i - full_starts);
    chunk_step<LEN, R, P, NC, EXACT, true, MPV>(st, chan, w, thr, init, one2, lo + (live ? v : 0), d,
                                           live ? n - v : 0, nan_slot);
    t += tstep;
    v0 += vstep;
    if (t >= radix) {
      t -= radix;
      v0 += vwrap;
    }
  }
  if constexpr (R > 1) {
    if (tail && rem > 0)
      run_positions<LEN, 1, P, NC, EXACT, MPV, LANES>(st, chan, w, thr, init, one2, lo + A * RD, rem, d, q32, r32,
                                                      invd, nan_slot, lane, false);
  }
}

// Position-paired step (single-kernel chunks, kinds 6 / 7): a lane holds two
// runs of R positions, run A at u0a + m*d and run B at u0b + m*d (m < R);
// FFMA2 lane .x computes run A's position r, lane .y run B's, both with the
// one kernel's weight (w, w) and the series values (xa[r + j], xb[r + j]) —
// a kernel slot that would idle beside a zero-weight partner does useful
// work instead.  The two windows are disjoint, so every element is loaded
// once, straight into its half of a pair slot.  Masking follows
// load_window_masked per run (a dead position's last tap reads the
// canonical NaN).  Per output the arithmetic is the one of chunk_step: same
// taps, same order, same rounding.
template <int LEN>
__device__ __forceinline__ float sp_load(const float* p, int e, int d, int nleft, const float* nan_slot, bool masked) {
  const float* a = p + e * d;
  if (masked && e >= LEN - 1) a = (e - (LEN - 1)) * d < nleft ? a : nan_slot;
  RK_CHK_READ(a, 4);
  return *a;
}

template <int LEN, int R, int NC, bool EXACT, bool MASKED, bool MPV = false>
__device__ __forceinline__ void chunk_step_sp(Pool<2, MPV>& st, const float* const (&chan)[NC],
                                              const float (&w)[NC][LEN], const float (&thr)[2], float2 init,
                                              float2 one2, int u0a, int u0b, int d, int nlefta, int nleftb,
                                              const float* nan_slot) {
  constexpr int C = (LEN - 1) / 2;
  constexpr int W = R + LEN - 1;
  float2 acc[1][R];
#pragma unroll
  for (int s = 0; s < NC; ++s) {
    const float* pa = chan[s] + (u0a - C * d);
    const float* pb = chan[s] + (u0b - C * d);
    auto tap = [&](int r, int j, float2 xq) {
      // the weight as a broadcast scalar
      const float2 w2 = make_float2(w[s][j], w[s][j]);
      if (EXACT) {
        if (s == 0 && j == 0)
          acc[0][r] = fmul2(xq, w2);  // RN(w*x) == RN(+0 + RN(w*x))
        else
          acc[0][r] = ffma2(fmul2(xq, w2), one2, acc[0][r]);
      } else {
        acc[0][r] = ffma2(xq, w2, (s == 0 && j == 0) ? init : acc[0][r]);
      }
    };
    if constexpr (NC == 1) {
      // anti-diagonal order: window entry q feeds taps j = q - r of the
      // positions r it covers and is dead afterwards, so only a few entries
      // are live at once (R up to 15 fits the registers); each output still
      // adds its taps in order j = 0 .. LEN-1
#pragma unroll
      for (int q = 0; q < W; ++q) {
        float2 xq;
        xq.x = sp_load<LEN>(pa, q, d, nlefta, nan_slot, MASKED);
        xq.y = sp_load<LEN>(pb, q, d, nleftb, nan_slot, MASKED);
#pragma unroll
        for (int r = 0; r < R; ++r)
          if (q - r >= 0 && q - r < LEN) tap(r, q - r, xq);
      }
    } else {
      float2 xp[W];
#pragma unroll
      for (int q = 0; q < W; ++q) {
        xp[q].x = sp_load<LEN>(pa, q, d, nlefta, nan_slot, MASKED);
        xp[q].y = sp_load<LEN>(pb, q, d, nleftb, nan_slot, MASKED);
      }
#pragma unroll
      for (int j = 0; j < LEN; ++j)
#pragma unroll
        for (int r = 0; r < R; ++r) tap(r, j, xp[r + j]);
    }
  }
  // slot 0 pools run A's positions, slot 1 run B's (same kernel)
  pool_update<R, 1, EXACT, false, MPV>(st, acc, thr, true, 0, d);
}

// run_positions for position-paired chunks: the lane map of run_positions
// with 64 run starts per step (starts base + lane and base + 32 + lane go
// to one lane's runs A and B).
template <int LEN, int R, int NC, bool EXACT, bool MPV = false>
__device__ __forceinline__ void run_positions_sp(Pool<2, MPV>& st, const float* const (&chan)[NC],
                                                 const float (&w)[NC][LEN], const float (&thr)[2], float2 init,
                                                 float2 one2, int lo, int n, int d, int q32, int r32, float invd,
                                                 const float* nan_slot, int lane, bool tail = false) {
  const int RD = R * d;
  const int A = n / RD;
  const int rem = n - A * RD;
  const int full_starts = A * d;
  const int starts = (R > 1 && tail) ? full_starts : full_starts + min(d, rem);  // see run_positions
  const int nfull = full_starts >> 6;
  int a = (int)((lane + 0.5f) * invd);
  int s = lane - a * d;
  int v0 = a * RD + s;
  const int dv = q32 * RD + r32;
  // advance a start by 32 (the existing incremental divmod)
  auto adv = [&](int& sv, int& vv) {
    sv += r32;
    vv += dv;
    if (sv >= d) {
      sv -= d;
      vv += RD - d;
    }
  };
#pragma unroll(kStepUnroll)
  for (int stp = 0; stp < nfull; ++stp) {
    int sb = s, vb = v0;
    adv(sb, vb);
    chunk_step_sp<LEN, R, NC, EXACT, false, MPV>(st, chan, w, thr, init, one2, lo + v0, lo + vb, d, n, n, nan_slot);
    s = sb;
    v0 = vb;
    adv(s, v0);
  }
  for (int base = nfull << 6; base < starts; base += 64) {
    int sb = s, vb = v0;
    adv(sb, vb);
    const bool la = base + lane < starts, lb = base + 32 + lane < starts;
    chunk_step_sp<LEN, R, NC, EXACT, true, MPV>(st, chan, w, thr, init, one2, lo + (la ? v0 : 0), lo + (lb ? vb : 0),
                                                d, la ? n - v0 : 0, lb ? n - vb : 0, nan_slot);
    s = sb;
    v0 = vb;
    adv(s, v0);
  }
  if constexpr (R > 1) {
    if (tail && rem > 0)
      run_positions_sp<LEN, 1, NC, EXACT, MPV>(st, chan, w, thr, init, one2, lo + A * RD, rem, d, q32, r32, invd,
                                               nan_slot, lane, false);
  }
}

// Finish a position-paired chunk: merge the two position slots (the
// CellAccumulator merge, engine.py:58-96), reduce over the warp, lane 0
// writes the kernel's features.
template <bool EXACT, class CH, bool MPV = false>
__device__ __forceinline__ void finish_chunk_sp(const CH& c, Pool<2, MPV>& st, float* __restrict__ orow, int fpk,
                                                int vec_out, int lane) {
  const unsigned tot = __reduce_add_sync(kFull, st.cnt[0] + st.cnt[1]);
  const float e = EXACT ? warp_max(fmaxf(st.ext[0], st.ext[1])) : warp_min(fminf(st.ext[0], st.ext[1]));
  float ps = 0.0f;
  if (MPV) {
    ps = st.ps[0].x + st.ps[0].y;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) ps += __shfl_xor_sync(kFull, ps, o);
  }
  if (lane == 0) {
    const float ppv = __fdiv_rn((float)tot, (float)c.n);  // == f32(RN64(count / l_out)), see finish_chunk
    const float mx = EXACT ? __fadd_rn(e, c.bias[0]) : -e;
    float* dst = orow + (int64_t)c.col[0] * fpk;
    RK_CHK_WRITE(dst, (MPV ? 3 : 2) * 4);
    if (vec_out) {
      *reinterpret_cast<float2*>(dst) = make_float2(ppv, mx);
    } else {
      dst[0] = ppv;
      dst[1] = mx;
    }
    if (MPV) dst[2] = tot ? __double2float_rn((double)(-ps) / (double)tot) : 0.0f;  // see finish_chunk
  }
}

// Run-time channel slots (NC = 0 kernels): the chunk's slot list and its
// weights ([slot][pair][tap] float2) live in the launch's parameter block;
// each step walks the slots in order — the reference's channel order — with
// one slot's weights loaded at a time (uniform registers) and one window.
template <int LEN, int R, int P, bool EXACT, bool MASKED, bool MPV = false>
__device__ __forceinline__ void chunk_step_dyn(Pool<2 * P, MPV>& st, const float* sx, const int* slots, int nc,
                                               const float2* wp, int S, const float (&thr)[2 * P],
                                               const float2 (&init)[P], float2 one2, int u0, int d, int nleft,
                                               const float* nan_slot) {
  float2 init_r[P][R];
#pragma unroll
  for (int p = 0; p < P; ++p)
#pragma unroll
    for (int r = 0; r < R; ++r) init_r[p][r] = init[p];
  float2 acc[P][R];
  {
    float xw[R + LEN - 1];
    if (MASKED)
      load_window_masked<LEN, R>(xw, sx + slots[0] * S, u0, d, nleft, nan_slot);
    else
      load_window<LEN, R>(xw, sx + slots[0] * S, u0, d);
    float2 w[P][LEN];
#pragma unroll
    for (int q = 0; q < P; ++q)
#pragma unroll
      for (int j = 0; j < LEN; ++j) w[q][j] = wp[q * LEN + j];
    accumulate<LEN, R, P, EXACT, true>(acc, w, xw, init_r, one2);
  }
  for (int s = 1; s < nc; ++s) {
    float xw[R + LEN - 1];
    if (MASKED)
      load_window_masked<LEN, R>(xw, sx + slots[s] * S, u0, d, nleft, nan_slot);
    else
      load_window<LEN, R>(xw, sx + slots[s] * S, u0, d);
    float2 w[P][LEN];
#pragma unroll
    for (int q = 0; q < P; ++q)
#pragma unroll
      for (int j = 0; j < LEN; ++j) w[q][j] = wp[(s * P + q) * LEN + j];
    accumulate<LEN, R, P, EXACT, false>(acc, w, xw, init_r, one2);
  }
  pool_update<R, P, EXACT, false, MPV>(st, acc, thr, true, 0, d);
}

// run_positions for run-time channel slots (same lane map).
template <int LEN, int R, int P, bool EXACT, bool MPV = false>
__device__ __forceinline__ void run_positions_dyn(Pool<2 * P, MPV>& st, const float* sx, const int* slots, int nc,
                                                  const float2* wp, int S, const float (&thr)[2 * P],
                                                  const float2 (&init)[P], float2 one2, int lo, int n, int d,
                                                  int q32, int r32, float invd, const float* nan_slot, int lane) {
  const int RD = R * d;
  const int A = n / RD;
  const int rem = n - A * RD;
  const int full_starts = A * d;
  const int starts = full_starts + min(d, rem);
  const int nfull = full_starts >> 5;
  int a = (int)((lane + 0.5f) * invd);
  int s = lane - a * d;
  int v0 = a * RD + s;
  const int dv = q32 * RD + r32;
  for (int stp = 0; stp < nfull; ++stp) {
    chunk_step_dyn<LEN, R, P, EXACT, false, MPV>(st, sx, slots, nc, wp, S, thr, init, one2, lo + v0, d, n,
                                                 nan_slot);
    s += r32;
    v0 += dv;
    if (s >= d) {
      s -= d;
      v0 += RD - d;
    }
  }
  for (int base = nfull << 5; base < starts; base += 32) {
    const bool live = base + lane < starts;
    chunk_step_dyn<LEN, R, P, EXACT, true, MPV>(st, sx, slots, nc, wp, S, thr, init, one2, lo + (live ? v0 : 0), d,
                                                live ? n - v0 : 0, nan_slot);
    s += r32;
    v0 += dv;
    if (s >= d) {
      s -= d;
      v0 += RD - d;
    }
  }
}

// Per-chunk constants of the pooling: exact thresholds, fast init pairs
// (-bias, moved through a shuffle so they live in vector registers and the
// first FFMA2 can read them next to a uniform-register weight).
template <int P, bool EXACT, class CH>
__device__ __forceinline__ void chunk_consts(const CH& c, float (&thr)[2 * P], float2 (&init)[P]) {
#pragma unroll
  for (int g = 0; g < 2 * P; ++g) thr[g] = EXACT ? c.thr[g] : 0.0f;
#pragma unroll
  for (int p = 0; p < P; ++p) {
    if (EXACT) {
      init[p] = make_float2(0.0f, 0.0f);
    } else {
      init[p].x = __shfl_sync(kFull, -c.bias[2 * p] + 0.0f, 0);
      init[p].y = __shfl_sync(kFull, -c.bias[2 * p + 1] + 0.0f, 0);
    }
  }
}

// Stage series rows [xs, xs + rows*L) into smem rows of stride S at offset
// H (negated for FAST).
template <bool EXACT>
__device__ __forceinline__ void stage_rows(float* __restrict__ smem, const float* __restrict__ xs, int rows, int L,
                                           int S, int H, int vec_in, int tid, int nthreads) {
  const float sg = EXACT ? 1.0f : -1.0f;
  if (vec_in) {
    const int L4 = L >> 2;
    for (int k = tid; k < rows * L4; k += nthreads) {
      const int row = k / L4, t = k - row * L4;
      const float4 v = __ldg(reinterpret_cast<const float4*>(xs + (int64_t)row * L) + t);
      *reinterpret_cast<float4*>(smem + row * S + H + 4 * t) = make_float4(sg * v.x, sg * v.y, sg * v.z, sg * v.w);
    }
  } else {
    for (int k = tid; k < rows * L; k += nthreads) {
      const int row = k / L, t = k - row * L;
      smem[row * S + H + t] = sg * __ldg(xs + k);
    }
  }
}

// One chunk with NC channel slots and register-resident weights (class
// kernel).
template <int LEN, int R, int P, int NC, bool EXACT>
__device__ __forceinline__ void run_chunk(const DevChunk& c, const float* __restrict__ sx,
                                          const float* __restrict__ weights, const int* __restrict__ chan_off,
                                          float* __restrict__ orow, int fpk, int vec_out, float one,
                                          const float* nan_slot, int lane) {
  constexpr int G = 2 * P;
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
  chunk_consts<P, EXACT>(c, thr, init);
  Pool<G> st;
  pool_init<G, EXACT>(st);
  run_positions<LEN, R, P, NC, EXACT>(st, chan, w, thr, init, make_float2(one, one), c.lo, c.n, c.d, c.q32,
                                      c.r32, c.invd, nan_slot, lane);
  finish_chunk<G, EXACT>(c, st, orow, fpk, vec_out, lane);
}

// Generic channel count (>= 3 slots): one kernel pair, one position per
// lane, slots looped at run time (the accumulator continues across slots in
// slot order, as the reference's channel loop).
template <int LEN, bool EXACT>
__device__ __forceinline__ void run_chunk_generic(const DevChunk& c, const float* __restrict__ sx,
                                                  const float* __restrict__ weights,
                                                  const int* __restrict__ chan_off, float* __restrict__ orow,
                                                  int fpk, int vec_out, float one, int lane) {
  constexpr int C = (LEN - 1) / 2;
  const float2* wp = reinterpret_cast<const float2*>(weights + c.wofs);
  float thr[2];
  float2 init[1];
  chunk_consts<1, EXACT>(c, thr, init);
  const float2 one2 = make_float2(one, one);
  Pool<2> st;
  pool_init<2, EXACT>(st);
  const int d = c.d, n = c.n, lo = c.lo, nc = c.nc;
  for (int t0 = 0; t0 < n; t0 += 32) {
    const int t = t0 + lane;
    const bool live = t < n;
    const int u = lo + (live ? t : 0);
    float2 acc[1][1];
    float2 init_r[1][1] = {{EXACT ? init[0] : (live ? init[0] : make_float2(INFINITY, INFINITY))}};
    for (int s = 0; s < nc; ++s) {
      const float* p = sx + __ldg(chan_off + c.chofs + s) + (u - C * d);
      float xw[LEN];
#pragma unroll
      for (int q = 0; q < LEN; ++q) xw[q] = p[q * d];
      float2 w[1][LEN];
#pragma unroll
      for (int j = 0; j < LEN; ++j) w[0][j] = __ldg(wp + s * LEN + j);
      if (s == 0)
        accumulate<LEN, 1, 1, EXACT, true>(acc, w, xw, init_r, one2);
      else
        accumulate<LEN, 1, 1, EXACT, false>(acc, w, xw, init_r, one2);
    }
    pool_update<1, 1, EXACT, EXACT>(st, acc, thr, live, 1, 1);
  }
  finish_chunk<2, EXACT>(c, st, orow, fpk, vec_out, lane);
}

// ---------------------------------------------------------------------------
// Class kernel: one launch per chunk class <LEN, R, NCK>.  Items are
// (group of series, block of this class's chunks); a CTA stages the series
// once per item and its warps pull chunks with a shared-memory counter;
// items are claimed dynamically.
template <int LEN, int R, int NCK, bool EXACT>
__global__ void __launch_bounds__(kThreads, kMinBlocks) rocket_class_kernel(const LaunchArgs a) {
  extern __shared__ __align__(16) float smem[];
  __shared__ int s_next;
  __shared__ int s_item;
  __shared__ float s_nan;  // the masked steps' dead-position source
  const int tid = threadIdx.x;
  const int lane = tid & 31;
  if (tid == 0) {
    s_nan = __int_as_float(0x7fffffff);
    RK_CHK_SET(smem, &s_nan, nullptr, nullptr, a.out, a.out + a.n_series * a.ld_out);
  }
  const int C = a.n_channels, L = a.l_series, H = a.halo, S = a.sstride;
  const int SPI = a.series_per_item;
  const int slot_floats = C * S;
  // Zero the halos once; only the interiors are rewritten per series.
  for (int k = tid; k < SPI * slot_floats; k += kThreads) {
    const int t = (k % slot_floats) % S;
    if (t < H || t >= H + L) smem[k] = 0.0f;
  }
  unsigned long long done = 0;
  while (true) {
    __syncthreads();  // every warp has left the previous item
    if (tid == 0) s_item = atomicAdd(a.item_counter, 1);
    __syncthreads();
    const int64_t item = s_item;
    if (item >= a.n_items) break;
    const int64_t group = item / a.n_blocks;
    const int blk = (int)(item - group * a.n_blocks);
    const int64_t series0 = group * SPI;
    const int64_t left = a.n_series - series0;
    const int ns = left < SPI ? (int)left : SPI;
    stage_rows<EXACT>(smem, a.x + series0 * (int64_t)C * L, ns * C, L, S, H, a.vec_in, tid, kThreads);
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
        run_chunk<LEN, R, 2, 1, EXACT>(c, sx, a.weights, a.chan_off, orow, a.fpk, a.vec_out, a.one, &s_nan, lane);
      else if (NCK == 1)
        run_chunk<LEN, R, 1, 2, EXACT>(c, sx, a.weights, a.chan_off, orow, a.fpk, a.vec_out, a.one, &s_nan, lane);
      else if (NCK == 3)
        run_chunk<LEN, R, 1, 1, EXACT>(c, sx, a.weights, a.chan_off, orow, a.fpk, a.vec_out, a.one, &s_nan, lane);
      else
        run_chunk_generic<LEN, EXACT>(c, sx, a.weights, a.chan_off, orow, a.fpk, a.vec_out, a.one, lane);
      done += (unsigned long long)c.nk * (unsigned long long)c.n;
    }
  }
  if (lane == 0 && done) atomicAdd(a.executed, done);
}

// ---------------------------------------------------------------------------
// Parameter-block launches (rocket_wide_kernel): the chunk descriptors and
// weights of one launch travel in the kernel's __grid_constant__ parameter
// block (<= 32 KB), so a warp-uniform chunk index lets ptxas keep the
// weights in uniform registers (LDCU) and FFMA2 read them as UR operands —
// ~80 vector registers instead of ~120, hence 24 resident warps per SM.
constexpr int kParamBytes = 32000;
struct float4_t {  // host-side storage of the parameter blob
  float x, y, z, w;
};

// WChunk.r32 bit 14: tail mode (complete runs at R, the remaining positions
// as an R = 1 map); the low bits hold 32 % d.  Kernels without the
// registers for the R = 1 path (kTailOK) ignore the flag and walk those
// chunks as partial runs: the same outputs in another order.
constexpr short kTailFlag = 0x4000;
// WChunk.r32 bit 13: run-major lane map (run_positions amap), log2 g in bits
// 8..10; bits 0..7 hold 32 % d (<= 32).
constexpr short kAMapFlag = 0x2000;
constexpr short kR32Mask = 0xFF;
__device__ __forceinline__ int chunk_amap(int r32) { return (r32 & kAMapFlag) ? ((r32 >> 8) & 7) : -1; }
struct __align__(16) WChunk {  // 80 bytes
  int d, lo, n, nk;
  int col[4];
  float bias[4];
  float thr[4];
  int ch[2];   // channel slots (smem offsets are ch * sstride)
  short q32;   // 32 / d (lane map, precomputed on the host)
  short r32;   // 32 % d
  float invd;  // 1 / d
};
static_assert(sizeof(WChunk) == 80, "WChunk layout");

struct WHeader {
  const float* x;
  float* out;
  unsigned long long* executed;
  int* item_counter;
  int64_t ld_out;
  int64_t n_series;
  int n_chunks;
  int l_series;
  int n_channels;
  int halo;
  int sstride;
  int fpk;
  int vec_out;
  int vec_in;
  float one;
  int wbytes;  // bytes of weights per chunk
  int spi;     // series per CTA item
  // series too long for shared memory (GMEM kernels): rows of sstride
  // floats with zero halos in a device scratch, and a canonical NaN there
  const float* xpad;
  const float* nanp;
};
constexpr int kBlobFloat4 = (kParamBytes - (int)sizeof(WHeader)) / 16;
struct WParams {
  WHeader h;
  float4 blob[kBlobFloat4];  // n_chunks WChunk, then n_chunks weight blocks
};

}  // namespace rk

// ---------------------------------------------------------------------------
// Cell kernel: one thread per (series, kernel) cell, the reference's loop
// verbatim (engine.py:157-188 and the MPV variant engine.py:202-247):
// positions ascending, channels then taps ascending, out-of-range taps
// skipped, RN(acc + RN(w*x)) without contraction, bias last, the positive
// sum accumulated in position order.  Used for precision "double" and for
// MPV (fpk = 3), where the ordered positive sum leaves no room for the
// reordered fast path.  Kernels are visited in a (length, channels, l_out)
// sorted order so a warp's threads run similar trip counts.
namespace rk {

struct __align__(16) CellKernel {
  int len, d, p, nc;
  int l_out, woff, choff, col;
};
static_assert(sizeof(CellKernel) == 32, "CellKernel layout");

struct CellArgs {
  const void* x;         // (n, C, L) of T, device
  void* out;             // row 0 of this launch
  int64_t ld_out;
  int64_t n_series;
  const CellKernel* kernels;
  const void* weights;   // T, reference layout (channel-major per kernel)
  const void* biases;    // T, per sorted kernel
  const int* chidx;
  unsigned long long* executed;
  int n_kernels;
  int l_series;
  int n_channels;
  int fpk;
  // staged variant (rocket_cellrow_kernel)
  int* item_counter;     // dynamic series scheduler (zeroed before the launch)
  int k_begin, k_end;    // sorted-kernel range of this launch (one length)
  int halo;              // zero halo per side of a staged row (elements)
  int sstride;           // elements per staged channel row
  const void* xpad;      // GMEM: zero-haloed rows of this launch's series
  float one;             // 1.0f, opaque to ptxas (FMUL2 + FFMA2 stay unfused)
};

template <typename T>
__device__ __forceinline__ T mul_rn(T a, T b);
template <>
__device__ __forceinline__ float mul_rn<float>(float a, float b) { return __fmul_rn(a, b); }
template <>
__device__ __forceinline__ double mul_rn<double>(double a, double b) { return __dmul_rn(a, b); }
template <typename T>
__device__ __forceinline__ T add_rn(T a, T b);
template <>
__device__ __forceinline__ float add_rn<float>(float a, float b) { return __fadd_rn(a, b); }
template <>
__device__ __forceinline__ double add_rn<double>(double a, double b) { return __dadd_rn(a, b); }
template <typename T>
__device__ __forceinline__ T from_double(double v);
template <>
__device__ __forceinline__ float from_double<float>(double v) { return __double2float_rn(v); }
template <>
__device__ __forceinline__ double from_double<double>(double v) { return v; }

template <typename T, bool MPV>
__global__ void __launch_bounds__(128) rocket_cell_kernel(const CellArgs a) {
  const int ks = blockIdx.x * blockDim.x + threadIdx.x;
  const bool live = ks < a.n_kernels;
  const CellKernel kd = live ? a.kernels[ks] : CellKernel{7, 1, 0, 1, 0, 0, 0, 0};
  const T* w = reinterpret_cast<const T*>(a.weights) + kd.woff;
  const T bias = live ? reinterpret_cast<const T*>(a.biases)[ks] : T(0);
  const int L = a.l_series, C = a.n_channels;
  unsigned long long done = 0;
  for (int64_t i = blockIdx.y; i < a.n_series; i += gridDim.y) {
    const T* xi = reinterpret_cast<const T*>(a.x) + i * (int64_t)C * L;
    int64_t count = 0;
    T running_max = -INFINITY;
    T psum = T(0);
    for (int t = 0; t < kd.l_out; ++t) {
      T acc = T(0);
      for (int c = 0; c < kd.nc; ++c) {
        const T* xc = xi + (int64_t)__ldg(a.chidx + kd.choff + c) * L;
        const T* wr = w + c * kd.len;
        for (int j = 0; j < kd.len; ++j) {
          const int idx = t - kd.p + j * kd.d;
          if (idx >= 0 && idx < L) acc = add_rn<T>(acc, mul_rn<T>(__ldg(wr + j), __ldg(xc + idx)));
        }
      }
      acc = add_rn<T>(acc, bias);
      if (acc > T(0)) {
        count += 1;
        if (MPV) psum = add_rn<T>(psum, acc);
      }
      if (acc > running_max) running_max = acc;
    }
    if (live) {
      T* o = reinterpret_cast<T*>(a.out) + i * a.ld_out + (int64_t)kd.col * a.fpk;
      o[0] = from_double<T>((double)count / (double)kd.l_out);
      o[1] = running_max;
      if (MPV) o[2] = count > 0 ? from_double<T>((double)psum / (double)count) : T(0);
      done += (unsigned long long)kd.l_out;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) done += __shfl_xor_sync(kFull, done, o);
  if ((threadIdx.x & 31) == 0 && done) atomicAdd(a.executed, done);
}

// Staged cell kernel: a CTA stages one series (all channels, zero halos)
// in shared memory; each warp takes 32 consecutive sorted kernels of one
// length LEN, one kernel per lane, and walks the positions in ascending
// order, B at a time (B independent accumulation chains).  Per position
// the arithmetic is the reference's: acc = +0, then RN(acc + RN(w*x)) over
// channels and taps in order, RN(acc + b), the positive sum in position
// order.  Out-of-range taps read the zero halo instead of being skipped:
// RN(w*0) is a signed zero and acc is never -0 (it starts at +0 and an RN
// sum is -0 only for -0 + -0), so acc + (+-0) == acc bit for bit.  Kernels
// are sorted by (length, channels, dilation, padding) so the lanes of a
// warp mostly read the same smem word (a broadcast) and run equal trip
// counts.
template <typename T, bool MPV, int LEN, int B, bool GMEM = false>
__global__ void __launch_bounds__(256) rocket_cellrow_kernel(const CellArgs a) {
  extern __shared__ __align__(16) unsigned char cell_smem[];
  T* xstage = reinterpret_cast<T*>(cell_smem);
  __shared__ int s_item, s_next;
  const int tid = threadIdx.x, lane = tid & 31;
  const int C = a.n_channels, L = a.l_series, H = a.halo, S = a.sstride;
  if (tid == 0)
    RK_CHK_SET(xstage, nullptr, a.xpad,
               GMEM ? reinterpret_cast<const T*>(a.xpad) + a.n_series * (int64_t)C * S : nullptr,
               a.out, reinterpret_cast<T*>(a.out) + a.n_series * a.ld_out);
  if constexpr (!GMEM) {
    for (int k = tid; k < C * S; k += blockDim.x) {
      const int t = k % S;
      if (t < H || t >= H + L) xstage[k] = T(0);
    }
  }
  const int ngroups = (a.k_end - a.k_begin + 31) / 32;
  const T* wts = reinterpret_cast<const T*>(a.weights);
  const T* bis = reinterpret_cast<const T*>(a.biases);
  unsigned long long done = 0;
  while (true) {
    __syncthreads();  // every warp has left the previous series
    if (tid == 0) {
      s_item = atomicAdd(a.item_counter, 1);
      s_next = 0;
    }
    __syncthreads();
    const int64_t i = s_item;
    if (i >= a.n_series) break;
    // GMEM: the series' zero-haloed rows are read from global memory (a
    // series too long for shared memory); otherwise staged here
    const T* xs = GMEM ? reinterpret_cast<const T*>(a.xpad) + i * (int64_t)C * S : xstage;
    if constexpr (!GMEM) {
      const T* xi = reinterpret_cast<const T*>(a.x) + i * (int64_t)C * L;
      for (int k = tid; k < C * L; k += blockDim.x) {
        const int c = k / L, t = k - c * L;
        xstage[c * S + H + t] = xi[k];
      }
      __syncthreads();
    }
    while (true) {
      int g = 0;
      if (lane == 0) g = atomicAdd(&s_next, 1);
      g = __shfl_sync(kFull, g, 0);
      if (g >= ngroups) break;
      const int ks = a.k_begin + g * 32 + lane;
      const bool live = ks < a.k_end;
      const CellKernel kd = a.kernels[live ? ks : a.k_begin + g * 32];
      const int lout = live ? kd.l_out : 0;
      const int span = __reduce_max_sync(kFull, lout);
      const T bias = bis[live ? ks : a.k_begin + g * 32];
      const T* wk = wts + kd.woff;
      T w0[LEN];  // slot-0 weights, kept for the whole walk
#pragma unroll
      for (int j = 0; j < LEN; ++j) w0[j] = wk[j];
      const T* x0 = xs + __ldg(a.chidx + kd.choff) * S + H - kd.p;
      int count = 0;
      T mx = T(-INFINITY), psum = T(0);
      for (int t0 = 0; t0 < span; t0 += B) {
        T acc[B];
#pragma unroll
        for (int b = 0; b < B; ++b) acc[b] = T(0);
        // dead positions (t >= l_out) re-read the last live window
        const int tb = min(t0, max(lout - B, 0));
#pragma unroll
        for (int j = 0; j < LEN; ++j) {
          const T* xp = x0 + tb + j * kd.d;
          RK_CHK_READ(xp, B * (int)sizeof(T));
#pragma unroll
          for (int b = 0; b < B; ++b) acc[b] = add_rn<T>(acc[b], mul_rn<T>(w0[j], xp[b]));
        }
        for (int c = 1; c < kd.nc; ++c) {
          const T* xc = xs + __ldg(a.chidx + kd.choff + c) * S + H - kd.p + tb;
          const T* wc = wk + c * LEN;
#pragma unroll
          for (int j = 0; j < LEN; ++j) {
            const T wj = wc[j];
            RK_CHK_READ(xc + j * kd.d, B * (int)sizeof(T));
#pragma unroll
            for (int b = 0; b < B; ++b) acc[b] = add_rn<T>(acc[b], mul_rn<T>(wj, xc[j * kd.d + b]));
          }
        }
        // position t0 + b is live iff t0 + b < lout; its accumulator is
        // acc[t0 + b - tb] (tb < t0 only in a lane's final, shifted block)
        const int shift = t0 - tb;
        auto pool = [&](T v) {
          v = add_rn<T>(v, bias);
          if (v > T(0)) {
            ++count;
            if (MPV) psum = add_rn<T>(psum, v);
          }
          if (v > mx) mx = v;
        };
        if (shift == 0) {
#pragma unroll
          for (int b = 0; b < B; ++b)
            if (t0 + b < lout) pool(acc[b]);
        } else {
#pragma unroll
          for (int b = 0; b < B; ++b) {
            const int q = b + shift;
            if (t0 + b < lout) {
              T v = acc[0];
#pragma unroll
              for (int r = 1; r < B; ++r) v = q == r ? acc[r] : v;
              pool(v);
            }
          }
        }
      }
      if (live) {
        T* o = reinterpret_cast<T*>(a.out) + i * a.ld_out + (int64_t)kd.col * a.fpk;
        RK_CHK_WRITE(o, (MPV ? 3 : 2) * (int)sizeof(T));
        o[0] = from_double<T>((double)count / (double)kd.l_out);
        o[1] = mx;
        if (MPV) o[2] = count > 0 ? from_double<T>((double)psum / (double)count) : T(0);
        done += (unsigned long long)kd.l_out;
      }
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) done += __shfl_xor_sync(kFull, done, o);
  if (lane == 0 && done) atomicAdd(a.executed, done);
}

// Position-paired cell kernel (precision "double" and exact MPV when two
// staged copies of a series fit): the reference's loop (engine.py:157-188,
// 202-247) with lane = kernel as in rocket_cellrow_kernel, but positions
// are evaluated in pairs (t, t + 1), t even: float32 taps as one FMUL2 and
// one FFMA2(prod, 1, acc) per pair — RN(acc + RN(w*x)) for each position,
// the same roundings in the same order — and the pair of series values
// (x[e], x[e + 1]) read with one 8-byte (16-byte for double) shared load.
// The series is staged twice, copy 1 shifted by one element, so that every
// pair is aligned in one of the copies: element e even -> copy 0 at e, e odd
// -> copy 1 at e - 1.  Per lane the copy depends only on the parity of
// (row offset + j*d), so two base pointers per channel slot (even and odd
// taps) replace any per-load selection.  MPV sums the positive outputs in
// position order (t, then t + 1), as the reference does.
#ifndef RK_CELLPAIR_NB32
#define RK_CELLPAIR_NB32 16
#endif
#ifndef RK_CELLPAIR_NB64
#define RK_CELLPAIR_NB64 8
#endif
template <typename T>
struct Pair;
template <>
struct Pair<float> {
  using V = float2;
};
template <>
struct Pair<double> {
  using V = double2;
};

template <typename T>
__device__ __forceinline__ typename Pair<T>::V pair_tap(typename Pair<T>::V acc, T w, typename Pair<T>::V x,
                                                       float2 one2, bool first);
template <>
__device__ __forceinline__ float2 pair_tap<float>(float2 acc, float w, float2 x, float2 one2, bool) {
  return ffma2(fmul2(x, make_float2(w, w)), one2, acc);  // RN(RN(w*x) * 1 + acc) == RN(acc + RN(w*x))
}
template <>
__device__ __forceinline__ double2 pair_tap<double>(double2 acc, double w, double2 x, float2, bool) {
  return make_double2(__dadd_rn(acc.x, __dmul_rn(w, x.x)), __dadd_rn(acc.y, __dmul_rn(w, x.y)));
}

// Positions per block: NB = 2 * NP pairs share each tap's address and
// weight (float32: 16, one address per eight 8-byte loads; float64: 8).
template <typename T>
__host__ __device__ constexpr int cellpair_nb() { return sizeof(T) == 4 ? RK_CELLPAIR_NB32 : RK_CELLPAIR_NB64; }
constexpr int kCellPairSlack = 32;  // elements past the two copies (dead-position reads reach <= NB past a row)

template <typename T, bool MPV, int LEN>
__global__ void __launch_bounds__(256) rocket_cellpair_kernel(const CellArgs a) {
  using V = typename Pair<T>::V;
  constexpr int NB = cellpair_nb<T>(), NP = NB / 2;
  extern __shared__ __align__(16) unsigned char cell_smem[];
  T* copy0 = reinterpret_cast<T*>(cell_smem);
  const int tid = threadIdx.x, lane = tid & 31;
  const int C = a.n_channels, L = a.l_series, H = a.halo, S = a.sstride;
  T* copy1 = copy0 + C * S;
  __shared__ int s_item, s_next;
  if (tid == 0)
    RK_CHK_SET(copy0, nullptr, nullptr, nullptr, a.out, reinterpret_cast<T*>(a.out) + a.n_series * a.ld_out);
  for (int k = tid; k < 2 * C * S + kCellPairSlack; k += blockDim.x) copy0[k] = T(0);
  const int ngroups = (a.k_end - a.k_begin + 31) / 32;
  const T* wts = reinterpret_cast<const T*>(a.weights);
  const T* bis = reinterpret_cast<const T*>(a.biases);
  const float2 one2 = make_float2(a.one, a.one);
  unsigned long long done = 0;
  while (true) {
    __syncthreads();  // every warp has left the previous series (and the zeroing is done)
    if (tid == 0) {
      s_item = atomicAdd(a.item_counter, 1);
      s_next = 0;
    }
    __syncthreads();
    const int64_t i = s_item;
    if (i >= a.n_series) break;
    const T* xi = reinterpret_cast<const T*>(a.x) + i * (int64_t)C * L;
    for (int k = tid; k < C * L; k += blockDim.x) {
      const int c = k / L, t = k - c * L;
      const T v = xi[k];
      copy0[c * S + H + t] = v;
      copy1[c * S + H + t - 1] = v;
    }
    __syncthreads();
    while (true) {
      int g = 0;
      if (lane == 0) g = atomicAdd(&s_next, 1);
      g = __shfl_sync(kFull, g, 0);
      if (g >= ngroups) break;
      const int ks = a.k_begin + g * 32 + lane;
      const bool live = ks < a.k_end;
      const CellKernel kd = a.kernels[live ? ks : a.k_begin + g * 32];
      const int lout = live ? kd.l_out : 0;
      const int span = __reduce_max_sync(kFull, lout);
      const T bias = bis[live ? ks : a.k_begin + g * 32];
      const T* wk = wts + kd.woff;
      const int d = kd.d;
      T w0[LEN];  // slot-0 weights, kept for the whole walk
#pragma unroll
      for (int j = 0; j < LEN; ++j) w0[j] = wk[j];
      // even taps start at parity(off), odd taps at parity(off + d)
      const int off0 = __ldg(a.chidx + kd.choff) * S + H - kd.p;
      const T* q00 = (off0 & 1) ? copy1 + off0 - 1 : copy0 + off0;
      const T* q01 = ((off0 + d) & 1) ? copy1 + off0 - 1 : copy0 + off0;
      int count = 0;
      T mx = T(-INFINITY), psum = T(0);
      for (int t0 = 0; t0 < span; t0 += NB) {
        // dead positions (t >= l_out) re-read the last live block; its
        // start is kept even (pairs (t, t + 1) stay aligned) and reads at
        // most one position past l_out (NB - 1 when l_out < NB; the
        // allocation ends in kCellPairSlack zeroed elements)
        int tb = min(t0, max(lout - NB, 0));
        tb += tb & 1;
        V acc[NP];  // acc = +0, then RN(acc + RN(w*x)) tap by tap (engine.py:172-179)
#pragma unroll
        for (int q = 0; q < NP; ++q) acc[q].x = acc[q].y = T(0);
#pragma unroll
        for (int j = 0; j < LEN; ++j) {
          const T* xp = ((j & 1) ? q01 : q00) + j * d + tb;
          RK_CHK_READ(xp, NB * (int)sizeof(T));
          RK_CHK(((uintptr_t)xp & (2 * sizeof(T) - 1)) == 0);
#pragma unroll
          for (int q = 0; q < NP; ++q)
            acc[q] = pair_tap<T>(acc[q], w0[j], *reinterpret_cast<const V*>(xp + 2 * q), one2, false);
        }
        for (int c = 1; c < kd.nc; ++c) {
          const int off = __ldg(a.chidx + kd.choff + c) * S + H - kd.p;
          const T* q0 = (off & 1) ? copy1 + off - 1 : copy0 + off;
          const T* q1 = ((off + d) & 1) ? copy1 + off - 1 : copy0 + off;
          const T* wc = wk + c * LEN;
#pragma unroll
          for (int j = 0; j < LEN; ++j) {
            const T* xp = ((j & 1) ? q1 : q0) + j * d + tb;
            RK_CHK_READ(xp, NB * (int)sizeof(T));
            RK_CHK(((uintptr_t)xp & (2 * sizeof(T) - 1)) == 0);
            const T wj = wc[j];
#pragma unroll
            for (int q = 0; q < NP; ++q)
              acc[q] = pair_tap<T>(acc[q], wj, *reinterpret_cast<const V*>(xp + 2 * q), one2, false);
          }
        }
        auto pool = [&](T v) {
          // branch-free: the count and the ordered positive sum advance
          // only on positive outputs (the sum's order is the position order)
          v = add_rn<T>(v, bias);
          const bool pos = v > T(0);
          count += pos ? 1 : 0;
          if (MPV) psum = pos ? add_rn<T>(psum, v) : psum;
          mx = v > mx ? v : mx;
        };
        const int shift = t0 - tb;
        if (shift == 0 && t0 + NB <= lout) {
#pragma unroll
          for (int q = 0; q < NP; ++q) {
            pool(acc[q].x);
            pool(acc[q].y);
          }
        } else {
#pragma unroll
          for (int b = 0; b < NB; ++b) {
            const int q = b + shift;
            if (t0 + b < lout) {
              T v = acc[0].x;
#pragma unroll
              for (int r = 1; r < NB; ++r) v = q == r ? ((r & 1) ? acc[r / 2].y : acc[r / 2].x) : v;
              pool(v);
            }
          }
        }
      }
      if (live) {
        T* o = reinterpret_cast<T*>(a.out) + i * a.ld_out + (int64_t)kd.col * a.fpk;
        RK_CHK_WRITE(o, (MPV ? 3 : 2) * (int)sizeof(T));
        o[0] = from_double<T>((double)count / (double)kd.l_out);
        o[1] = mx;
        if (MPV) o[2] = count > 0 ? from_double<T>((double)psum / (double)count) : T(0);
        done += (unsigned long long)kd.l_out;
      }
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) done += __shfl_xor_sync(kFull, done, o);
  if (lane == 0 && done) atomicAdd(a.executed, done);
}

}  // namespace rk

// ---------------------------------------------------------------------------
// Wide kernel (every chunk class with <= 2 channel slots): W warps per CTA
// share one staged series and claim whole chunks of the launch's parameter
// block from a shared counter; CTAs claim series from a global counter.  The
// claimed chunk index is passed through a warp REDUX, whose result lives in
// a uniform register, so ptxas loads the chunk's descriptor and weights with
// LDCU into uniform registers and FFMA2 reads the weights as UR operands.
// CTAs x W is sized for 24 warps per SM (shared memory permitting).
namespace rk {

#ifndef RK_WIDE_WARPS
#define RK_WIDE_WARPS 24  // resident warps per SM the wide kernel is built for (~80 registers)
#endif
constexpr int kWideMaxWarps = RK_WIDE_WARPS;

// 1-D TMA (cp.async.bulk) staging of whole series rows, completed on an
// mbarrier.
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned bar, unsigned phase) {
  asm volatile(
      "{\n\t.reg .pred done;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 done, [%0], %1;\n\t"
      "@!done bra WAIT_%=;\n\t}" ::"r"(bar),
      "r"(phase)
      : "memory");
}
__device__ __forceinline__ void tma_row(unsigned dst, const void* src, unsigned bytes, unsigned bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(bar)
               : "memory");
}

template <int LEN, int R, int P, int NC, bool EXACT, bool MPV = false, bool GMEM = false, int LG = 32,
          bool SP = false>
__global__ void __launch_bounds__(32 * kWideMaxWarps, 1) rocket_wide_kernel(const __grid_constant__ WParams p) {
  extern __shared__ __align__(16) float smem[];
  __shared__ int s_item;
  __shared__ int s_next;
  __shared__ float s_nan;  // the masked steps' dead-position source
  __shared__ __align__(8) unsigned long long s_bar;  // TMA staging barrier
  asm volatile("griddepcontrol.launch_dependents;");
  const int tid = threadIdx.x, lane = tid & 31;
  const unsigned bar = smem_u32(&s_bar);
  unsigned phase = 0;
  if (tid == 0) {
    s_nan = __int_as_float(0x7fffffff);
    if (!GMEM && p.h.vec_in) mbar_init(bar, 1);
    RK_CHK_SET(smem, GMEM ? (const void*)p.h.nanp : (const void*)&s_nan, p.h.xpad, GMEM ? p.h.nanp + 1 : nullptr,
               p.h.out, p.h.out + p.h.n_series * p.h.ld_out);
  }
  const int C = p.h.n_channels, L = p.h.l_series, H = p.h.halo, S = p.h.sstride;
  const int SPI = p.h.spi;
  const int slot = C * S;
  if constexpr (!GMEM) {
    for (int k = tid; k < SPI * slot; k += blockDim.x) {
      const int t = (k % slot) % S;
      if (t < H || t >= H + L) smem[k] = 0.0f;
    }
  }
  // GMEM: the windows are read from the zero-haloed rows in global memory
  // (L1 / L2 resident) instead of a staged copy
  const float* nanp = GMEM ? p.h.nanp : &s_nan;
  const WChunk* chunks = reinterpret_cast<const WChunk*>(p.blob);
  // tail mode support (see kTailFlag): the fast-MPV lane-group kernels at
  // R >= 11 keep too many partial sums live for the R = 1 path and walk tail
  // chunks as partial runs instead (the same outputs in another order)
  constexpr bool kTailOK = !MPV || LG == 32 || R <= 9;
  const char* wbase = reinterpret_cast<const char*>(p.blob) + (size_t)p.h.n_chunks * sizeof(WChunk);
  const float2 one2 = make_float2(p.h.one, p.h.one);
  unsigned long long done = 0;
  while (true) {
    __syncthreads();  // every warp has left the previous item
    if (tid == 0) {
      s_item = atomicAdd(p.h.item_counter, 1);
      s_next = 0;
    }
    __syncthreads();
    const int64_t series0 = (int64_t)s_item * SPI;
    if (series0 >= p.h.n_series) break;
    const int64_t left = p.h.n_series - series0;
    const int ns = left < SPI ? (int)left : SPI;
    // Stage the item's rows unchanged (FAST negates the weights instead of
    // the series): one bulk copy per row when rows are 16-byte aligned,
    // else a cooperative copy.
    const float* sbase = GMEM ? p.h.xpad + series0 * slot : smem;
    if (GMEM) {
    } else if (p.h.vec_in) {
      if (tid == 0) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // prior generic reads of the buffer
        const unsigned row_bytes = (unsigned)L * 4u;
        mbar_expect_tx(bar, row_bytes * (unsigned)(ns * C));
        const float* src = p.h.x + series0 * C * L;
        for (int r = 0; r < ns * C; ++r) {
          RK_CHK_READ(smem + r * S + H, (int)row_bytes);
          RK_CHK(series0 + (r / C) < p.h.n_series);
          tma_row(smem_u32(smem + r * S + H), src + (int64_t)r * L, row_bytes, bar);
        }
      }
      mbar_wait(bar, phase);
      phase ^= 1;
    } else {
      stage_rows<true>(smem, p.h.x + series0 * C * L, ns * C, L, S, H, 0, tid, blockDim.x);
      __syncthreads();
    }
    while (true) {
      int ci = 0;
      if (lane == 0) ci = atomicAdd(&s_next, 1);
      // REDUX result lands in a uniform register: the chunk index is
      // warp-uniform for ptxas from here on
      ci = __reduce_max_sync(kFull, __shfl_sync(kFull, ci, 0));
      if (ci >= p.h.n_chunks) break;
      const WChunk& c = chunks[ci];
      float thr[2 * P];
      float2 init[P];
      chunk_consts<P, EXACT>(c, thr, init);
      if constexpr (NC == 0) {
        // run-time slots: ch[0] = byte offset of the chunk's weights in the
        // block, ch[1] = slot count; the slot list follows the weights
        const int nc = c.ch[1];
        const float2* wp = reinterpret_cast<const float2*>(reinterpret_cast<const char*>(p.blob) + c.ch[0]);
        const int* slots = reinterpret_cast<const int*>(wp + nc * P * LEN);
        for (int si = 0; si < ns; ++si) {
          Pool<2 * P, MPV> st;
          pool_init<2 * P, EXACT, MPV>(st);
          run_positions_dyn<LEN, R, P, EXACT, MPV>(st, sbase + si * slot + H, slots, nc, wp, S, thr, init, one2,
                                                   c.lo, c.n, c.d, c.q32, c.r32, c.invd, nanp, lane);
          finish_chunk<2 * P, EXACT, WChunk, MPV>(c, st, p.h.out + (series0 + si) * p.h.ld_out, p.h.fpk,
                                                  p.h.vec_out, lane);
          done += (unsigned long long)c.nk * (unsigned long long)c.n;
        }
      } else {
        const float2* wp = reinterpret_cast<const float2*>(wbase + (size_t)ci * p.h.wbytes);
        if constexpr (SP) {
          // position-paired single-kernel chunk: the host packed (w, w)
          static_assert(P == 1 && LG == 32 && !GMEM, "position-paired chunks: one kernel, full warp, staged series");
          float ws[NC][LEN];
#pragma unroll
          for (int s = 0; s < NC; ++s)
#pragma unroll
            for (int j = 0; j < LEN; ++j) ws[s][j] = wp[s * LEN + j].x;
          const float thr2[2] = {thr[0], thr[0]};
          const float2 init2 = make_float2(init[0].x, init[0].x);
          for (int si = 0; si < ns; ++si) {
            const float* sx = sbase + si * slot + H;
            const float* chan[NC];
#pragma unroll
            for (int s = 0; s < NC; ++s) chan[s] = sx + c.ch[s] * S;
            Pool<2, MPV> st;
            pool_init<2, EXACT, MPV>(st);
            run_positions_sp<LEN, R, NC, EXACT, MPV>(st, chan, ws, thr2, init2, one2, c.lo, c.n, c.d, c.q32,
                                                     c.r32 & kR32Mask, c.invd, nanp, lane,
                                                     kTailOK && (c.r32 & kTailFlag) != 0);
            finish_chunk_sp<EXACT, WChunk, MPV>(c, st, p.h.out + (series0 + si) * p.h.ld_out, p.h.fpk, p.h.vec_out,
                                                lane);
            done += (unsigned long long)c.n;
          }
          continue;
        }
        float2 w[NC][P][LEN];
#pragma unroll
        for (int s = 0; s < NC; ++s)
#pragma unroll
          for (int q = 0; q < P; ++q)
#pragma unroll
            for (int j = 0; j < LEN; ++j) w[s][q][j] = wp[(s * P + q) * LEN + j];
        if constexpr (LG < 32) {
          // lane-group chunks: 32 / LG series per pass, LG lanes each
          // (finer step granularity for short position ranges); groups past
          // the last series shadow it and write nothing
          static_assert(!GMEM && !(MPV && EXACT), "lane-group chunks: staged series; MPV in fast mode");
          constexpr int NG = 32 / LG;
          constexpr int kLogLG = LG == 16 ? 4 : LG == 8 ? 3 : 2;
          const int grp = lane >> kLogLG, hl = lane & (LG - 1);
          const int qg = c.q32 >> (5 - kLogLG), rg = LG - qg * c.d;  // LG / d, LG % d
          for (int si = 0; si < ns; si += NG) {
            const int sj = min(si + grp, ns - 1);
            const float* sx = sbase + sj * slot + H;
            const float* chan[NC];
#pragma unroll
            for (int s = 0; s < NC; ++s) chan[s] = sx + c.ch[s] * S;
            Pool<2 * P, MPV> st;
            pool_init<2 * P, EXACT, MPV>(st);
            run_positions<LEN, R, P, NC, EXACT, MPV, LG>(st, chan, w, thr, init, one2, c.lo, c.n, c.d, qg, rg,
                                                         c.invd, nanp, hl, kTailOK && (c.r32 & kTailFlag) != 0,
                                                         chunk_amap(c.r32));
            float* orow0 = p.h.out + (series0 + si) * p.h.ld_out;
            float* orow = orow0;
#pragma unroll
            for (int g = 1; g < NG; ++g)
              if (grp == g) orow = si + g < ns ? orow0 + g * p.h.ld_out : nullptr;
            finish_chunk_group<2 * P, EXACT, WChunk, MPV, LG>(c, st, orow, p.h.fpk, p.h.vec_out, lane);
            done += (unsigned long long)c.nk * (unsigned long long)c.n * (unsigned)min(NG, ns - si);
          }
          continue;
        }
        // the chunk's weights serve every staged series of the item
        for (int si = 0; si < ns; ++si) {
          const float* sx = sbase + si * slot + H;
          const float* chan[NC];
#pragma unroll
          for (int s = 0; s < NC; ++s) chan[s] = sx + c.ch[s] * S;
          Pool<2 * P, MPV> st;
          pool_init<2 * P, EXACT, MPV>(st);
          run_positions<LEN, R, P, NC, EXACT, MPV>(st, chan, w, thr, init, one2, c.lo, c.n, c.d, c.q32,
                                                   c.r32 & kR32Mask, c.invd, nanp, lane,
                                                   kTailOK && (c.r32 & kTailFlag) != 0, chunk_amap(c.r32));
          finish_chunk<2 * P, EXACT, WChunk, MPV>(c, st, p.h.out + (series0 + si) * p.h.ld_out, p.h.fpk,
                                                  p.h.vec_out, lane);
          done += (unsigned long long)c.nk * (unsigned long long)c.n;
        }
      }
    }
  }
  if (lane == 0 && done) atomicAdd(p.h.executed, done);
}

}  // namespace rk
