// kernels_len.cu — instantiates the kernels of one tap length (RK_LEN) and
// one positions-per-lane class (RK_RI) and exports the table filler declared
// in kernel_tables.h; the 3 x 8 units build in parallel.
#include "kernel_tables.h"

#if !defined(RK_LEN) || !defined(RK_RI)
#error "compile with -DRK_LEN=7|9|11 -DRK_RI=0..7"
#endif

namespace {
constexpr int kLenIdx = (RK_LEN - 7) / 2;

// Exact mode never runs R above kExactRMax (exec_cls caps it), so those
// exact variants are not instantiated.
template <int RI, int NCK>
void fill_class(rk::KernelFn* t, int cls) {
  constexpr int R = rk::r_of(RI);
  t[2 * cls + 0] = rk::rocket_class_kernel<RK_LEN, R, NCK, false>;
  if constexpr (R <= rk::kExactRMax) t[2 * cls + 1] = rk::rocket_class_kernel<RK_LEN, R, NCK, true>;
}

template <int RI, int P, int NC>
void fill_wide(rk::WarpFn* wide, rk::WarpFn* mpv, int cls) {
  constexpr int R = rk::r_of(RI);
  wide[2 * cls + 0] = rk::rocket_wide_kernel<RK_LEN, R, P, NC, false>;
  if constexpr (R <= rk::kExactRMax) {
    wide[2 * cls + 1] = rk::rocket_wide_kernel<RK_LEN, R, P, NC, true>;
    mpv[cls] = rk::rocket_wide_kernel<RK_LEN, R, P, NC, false, true>;
  }
}

// lane-group chunks (single channel; LG = 16 half-warp, 8 quarter-warp):
// PPV/MAX kernels and the fast MPV kernel
template <int RI, int P, int LG>
void fill_group(rk::WarpFn* wide, rk::WarpFn* mpv, int cls) {
  constexpr int R = rk::r_of(RI);
  wide[2 * cls + 0] = rk::rocket_wide_kernel<RK_LEN, R, P, 1, false, false, false, LG>;
  if constexpr (R <= rk::kExactRMax) {
    wide[2 * cls + 1] = rk::rocket_wide_kernel<RK_LEN, R, P, 1, true, false, false, LG>;
    mpv[cls] = rk::rocket_wide_kernel<RK_LEN, R, P, 1, false, true, false, LG>;
  }
}

// position-paired single-kernel chunks (kinds 6 / 7): PPV/MAX and fast MPV
template <int RI, int NC>
void fill_sp(rk::WarpFn* wide, rk::WarpFn* mpv, int cls) {
  constexpr int R = rk::r_of(RI);
  if constexpr (R <= rk::sp_rmax(NC, RK_LEN)) {
    wide[2 * cls + 0] = rk::rocket_wide_kernel<RK_LEN, R, 1, NC, false, false, false, 32, true>;
    wide[2 * cls + 1] = rk::rocket_wide_kernel<RK_LEN, R, 1, NC, true, false, false, 32, true>;
    mpv[cls] = rk::rocket_wide_kernel<RK_LEN, R, 1, NC, false, true, false, 32, true>;
  }
}

// GMEM variants: every chunk uses the run-time slot layout; 2-pair chunks
// at R <= 5, 1-pair chunks at any R — within registers.
template <int RI, int P>
void fill_gmem(rk::WarpFn* g, int cls) {
  constexpr int R = rk::r_of(RI);
  if constexpr (P == 1 || RI <= 2) {
    g[2 * cls + 0] = rk::rocket_wide_kernel<RK_LEN, R, P, 0, false, false, true>;
    if constexpr (R <= rk::kExactRMax) g[2 * cls + 1] = rk::rocket_wide_kernel<RK_LEN, R, P, 0, true, false, true>;
  }
}

template <int RI>
void fill_r(rk::KernelFn* ct, rk::WarpFn* dt, rk::WarpFn* mt, rk::WarpFn* gt) {
  constexpr int R = rk::r_of(RI);
  const int base = (kLenIdx * rk::kNumR + RI) * rk::kNumNck;
  fill_class<RI, 0>(ct, base + 0);
  fill_class<RI, 1>(ct, base + 1);
  fill_class<RI, 3>(ct, base + 3);
  if constexpr (R == 1) fill_class<RI, 2>(ct, base + 2);  // generic channels: 1 position per lane
  fill_wide<RI, 2, 1>(dt, mt, base + 0);
  fill_wide<RI, 1, 2>(dt, mt, base + 1);
  fill_wide<RI, 1, 0>(dt, mt, base + 2);
  fill_wide<RI, 1, 1>(dt, mt, base + 3);
  fill_group<RI, 2, 16>(dt, mt, base + 4);
  fill_group<RI, 1, 16>(dt, mt, base + 5);
  fill_group<RI, 2, 8>(dt, mt, base + 8);
  fill_group<RI, 1, 8>(dt, mt, base + 9);
  fill_group<RI, 2, 4>(dt, mt, base + 10);
  fill_group<RI, 1, 4>(dt, mt, base + 11);
  fill_sp<RI, 1>(dt, mt, base + 6);
  fill_sp<RI, 2>(dt, mt, base + 7);
  fill_gmem<RI, 2>(gt, base + 0);
  fill_gmem<RI, 1>(gt, base + 1);
  fill_gmem<RI, 1>(gt, base + 2);
  fill_gmem<RI, 1>(gt, base + 3);
}
}  // namespace

#define RK_CAT2(a, b, c) a##b##_##c
#define RK_CAT(a, b, c) RK_CAT2(a, b, c)

void RK_CAT(rk_fill_tables_, RK_LEN, RK_RI)(rk::KernelFn* ct, rk::WarpFn* dt, rk::WarpFn* mt, rk::WarpFn* gt) {
  if constexpr (RK_RI < rk::kNumR) fill_r<RK_RI>(ct, dt, mt, gt);
}
