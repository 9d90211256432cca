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

// Fill the (class, mode) slots of length LEN: class kernels into cls_tab,
// wide kernels into wide_tab (index 2 * cls + exact), and the fast-mode MPV
// wide kernels into mpv_tab (index cls; R capped like exact mode).
// gmem_tab (index 2 * cls + exact): the variants reading series rows from
// global memory, for series longer than shared memory holds.
void rk_fill_tables_7(rk::KernelFn* cls_tab, rk::WarpFn* wide_tab, rk::WarpFn* mpv_tab, rk::WarpFn* gmem_tab);
void rk_fill_tables_9(rk::KernelFn* cls_tab, rk::WarpFn* wide_tab, rk::WarpFn* mpv_tab, rk::WarpFn* gmem_tab);
void rk_fill_tables_11(rk::KernelFn* cls_tab, rk::WarpFn* wide_tab, rk::WarpFn* mpv_tab, rk::WarpFn* gmem_tab);
