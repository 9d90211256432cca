// kernel_tables.h — per-length kernel instantiation tables.  Each
// rk_fill_tables_<LEN> lives in its own translation unit (kernels_len.cu
// compiled with -DRK_LEN=<LEN>) so the 100+ template instantiations build in
// parallel; the host runtime (rocket_b200.cu) launches them through these
// function pointers.
#pragma once
#include "transform_kernel.cuh"

namespace rk {
using KernelFn = void (*)(const LaunchArgs);
using WarpFn = void (*)(const WParams);
}  // namespace rk

// Fill the (class, mode) slots of length LEN and R class RI: class kernels
// into cls_tab, wide kernels into wide_tab (index 2 * cls + exact), the
// fast-mode MPV wide kernels into mpv_tab (index cls), and the variants
// reading series rows from global memory (series longer than shared memory
// holds) into gmem_tab (index 2 * cls + exact).
#define RK_FILL_DECL(L, R)                                                                               \
  void rk_fill_tables_##L##_##R(rk::KernelFn* cls_tab, rk::WarpFn* wide_tab, rk::WarpFn* mpv_tab, \
                                rk::WarpFn* gmem_tab);
#define RK_FILL_DECL_L(L) \
  RK_FILL_DECL(L, 0) RK_FILL_DECL(L, 1) RK_FILL_DECL(L, 2) RK_FILL_DECL(L, 3) RK_FILL_DECL(L, 4) \
  RK_FILL_DECL(L, 5) RK_FILL_DECL(L, 6) RK_FILL_DECL(L, 7)
RK_FILL_DECL_L(7)
RK_FILL_DECL_L(9)
RK_FILL_DECL_L(11)
