/*
 * rocket_b200.h — C ABI of the B200-native ROCKET transform.
 *
 * This is the drop-in boundary for the reference's hot path: the numba
 * kernel call in gridrocket's engine
 *
 *     kernel(x[start:start+count], bank.lengths, bank.dilations, bank.paddings,
 *            biases, wflat, bank.weight_offsets, bank.channel_indices,
 *            bank.channel_offsets, bank.channel_counts,
 *            limits.workers_per_cell, fpk, out, row0 + start) -> executed
 *
 * (/root/reference/pkg/src/gridrocket/engine.py:280-295, selecting
 * _run_batch at engine.py:148-190).  Every entry point takes plain pointers
 * and sizes; no torch or numpy types cross this boundary.  All functions
 * return 0 on success and a nonzero RK_ERR_* code on failure; the message of
 * the last failure on the calling thread is available from rk_last_error().
 *
 * Pointers named "x" and "out" may be host (pageable or pinned) or device
 * memory; the library detects which with cudaPointerGetAttributes and moves
 * data as needed.  Bank parameters are always host pointers.
 */
#ifndef ROCKET_B200_H
#define ROCKET_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RK_ABI_VERSION 2

/* Error codes.  RK_ERR_CAPACITY mirrors gridrocket.CapacityError
 * (engine.py:30-31); RK_ERR_INVALID mirrors the ValueError raised by
 * _check_shapes / KernelBank.validate (engine.py:252-268, kernels.py:101-125). */
#define RK_OK 0
#define RK_ERR_INVALID 1
#define RK_ERR_CAPACITY 2
#define RK_ERR_CUDA 3
#define RK_ERR_UNSUPPORTED 4
#define RK_ERR_NO_DEVICE 5

/* Arithmetic modes.
 * RK_MODE_EXACT: every tap is RN(acc + RN(w*x)), channels ascending, taps
 *   ascending, bias after the last tap — bit-identical to the reference's
 *   single-precision engine (engine.py:172-180, reference.py:1-17).
 * RK_MODE_FAST: fused multiply-add (FFMA2), bias folded into the
 *   accumulator; within the north-star tolerance (MAX 1e-5 relative, PPV
 *   exact except for outputs within 1e-6 of zero). */
#define RK_MODE_EXACT 0
#define RK_MODE_FAST 1

/* Element types of x and out (engine.py's precision "single" / "double",
 * features.py:16-24). */
#define RK_DTYPE_F32 0
#define RK_DTYPE_F64 1

typedef struct rk_bank_s* rk_bank_t;

/* Summary of a device bank (the dilation-grouped layout). */
typedef struct rk_bank_info_s {
  int64_t n_kernels;
  int32_t n_channels;
  int32_t l_series;
  int32_t n_groups;     /* distinct (length, dilation, padding, channel set) */
  int32_t n_chunks;     /* warp work units (<= 4 kernels of one group) */
  int32_t halo;         /* zero halo per side in the staged series (floats) */
  int32_t smem_bytes;   /* dynamic shared memory per CTA */
  int64_t positions_per_series; /* sum_k l_out_k == engine.total_positions */
  int64_t useful_flops_per_series; /* sum_k 2*in-range taps + l_out_k */
  int64_t device_bytes; /* device memory held by the bank */
  int32_t device;
  int32_t n_launches;   /* kernel launches per float32 transform */
  int32_t path;         /* 1: wide kernel (parameter-block weights in
                           uniform registers, series staged in shared
                           memory); 2: wide kernel reading series rows from
                           global memory (series too long for shared
                           memory); 0: class kernel (RK_NO_WIDE_PATH) */
  int32_t ctas_per_sm;  /* resident CTAs per SM on the wide path */
  int32_t n_half_chunks; /* chunks laid out as half-warp chunks (two series
                            per 16-lane pass) in the fast-mode layout */
  int32_t n_paired_chunks; /* single-kernel chunks run position-paired (the
                               two FFMA2 lanes on two positions of the kernel) */
  int32_t n_quarter_chunks; /* chunks laid out as quarter-warp chunks (four
                               series per 8-lane pass) in the fast-mode layout */
  int32_t n_eighth_chunks;  /* chunks laid out as eighth-warp chunks (eight
                               series per 4-lane pass) in the fast-mode layout */
  int32_t n_runmajor_chunks; /* chunks whose run starts are dealt run-major
                                (fewer shared-memory bank conflicts) */
} rk_bank_info_t;

/* ABI version (RK_ABI_VERSION) and the thread-local last error message. */
int rk_abi_version(void);
const char* rk_last_error(void);

/* Number of visible CUDA devices (0 on a host without a GPU). */
int rk_device_count(int32_t* count);

/* Build the device bank once per KernelBank.  The arrays are the columnar
 * KernelBank fields (kernels.py:51-99) with weights and biases already cast
 * to float32 as in engine._run_range (engine.py:275-276); weight_offsets and
 * channel_offsets are KernelBank.weight_offsets / channel_offsets
 * (kernels.py:84-88).  Replaces the per-batch argument list of the numba
 * call at engine.py:280-295.  A series whose zero-haloed rows do not fit in
 * one CTA's shared memory is read from global memory instead (slower, no
 * length limit; rk_bank_info_t.path == 2). */
int rk_bank_create(int64_t n_kernels, int32_t n_channels, int32_t l_series,
                   const int32_t* lengths, const int32_t* dilations,
                   const int32_t* paddings, const float* biases,
                   const float* weights, const int64_t* weight_offsets,
                   const int32_t* channel_indices,
                   const int64_t* channel_offsets,
                   const int32_t* channel_counts, int32_t device,
                   rk_bank_t* bank);
int rk_bank_destroy(rk_bank_t bank);

/* Attach the float64 parameters (KernelBank.biases / .weights, uncast) for
 * precision "double" transforms (engine.py:274-276 casts to the compute
 * dtype, which for "double" is the identity). */
int rk_bank_attach_f64(rk_bank_t bank, const double* biases, const double* weights);
int rk_bank_info(rk_bank_t bank, rk_bank_info_t* info);

/* Transform n_series series x[(n_series, n_channels, l_series), C-contiguous,
 * element type dtype] with every kernel of the bank and write rows
 * [row0, row0 + n_series) of out (same element type, row stride ld_out
 * elements) in the reference layout: out[row, k*fpk] = ppv_k,
 * out[row, k*fpk + 1] = max_k and, for fpk == 3, out[row, k*fpk + 2] = mpv_k
 * (features.py:1-5, engine.py:186-188, 236-247).  float32 runs the FFMA2
 * kernels in either mode, except fpk == 3 in RK_MODE_EXACT; float64, and
 * fpk == 3 in RK_MODE_EXACT, run the cell kernels (the reference loop
 * order, bit-identical).  Fast-mode MPV sums the positive outputs per lane
 * and then across the warp (within 1e-5 relative).  x and out may be host or
 * device pointers.  stream is a
 * cudaStream_t (NULL = the caller's default stream: the transform runs on the
 * library's per-device stream, ordered after the work already queued on the
 * default stream and before the work queued there later); for device x and
 * out the call is asynchronous on that stream, otherwise it returns after
 * the features are in out.  *executed (may be NULL) receives the number of
 * dot-product positions evaluated, counted on the device; it equals
 * engine.expected_dot_products (engine.py:137-145). */
int rk_transform(rk_bank_t bank, const void* x, int32_t dtype, int64_t n_series,
                 void* out, int64_t ld_out, int64_t row0, int32_t fpk,
                 int32_t mode, void* stream, int64_t* executed);
/* rk_transform with dtype RK_DTYPE_F32. */
int rk_transform_f32(rk_bank_t bank, const float* x, int64_t n_series,
                     float* out, int64_t ld_out, int64_t row0, int32_t fpk,
                     int32_t mode, void* stream, int64_t* executed);

/* Stateless mirror of the numba entry point _run_batch
 * (engine.py:148-190; called at engine.py:280-295): same arguments in the
 * same order plus explicit sizes, returns the executed position count
 * (>= 0) or -(RK_ERR_*) on failure.  The device bank is built on first use
 * and cached by the identity and content of the bank arrays.  x and out are
 * host pointers (the numpy arrays the engine passes); workers_per_cell is
 * accepted for signature parity and, as in the reference, cannot change
 * the result.  fpk 3 adds MPV (_run_batch_mpv, engine.py:193-249).  Uses
 * RK_MODE_EXACT so results are byte-identical. */
int64_t rk_run_batch_f32(const float* x, int64_t n_instances,
                         int32_t n_channels, int32_t l_series,
                         const int32_t* lengths, const int32_t* dilations,
                         const int32_t* paddings, const float* biases,
                         const float* wflat, const int64_t* woff,
                         const int32_t* chidx, const int64_t* choff,
                         const int32_t* chcnt, int64_t n_kernels,
                         int32_t workers, int32_t fpk, float* out,
                         int64_t ld_out, int64_t row0);

/* The same for precision "double" (the float64 kernel the reference's
 * engine runs for precision="double", engine.py:274-276). */
int64_t rk_run_batch_f64(const double* x, int64_t n_instances,
                         int32_t n_channels, int32_t l_series,
                         const int32_t* lengths, const int32_t* dilations,
                         const int32_t* paddings, const double* biases,
                         const double* wflat, const int64_t* woff,
                         const int32_t* chidx, const int64_t* choff,
                         const int32_t* chcnt, int64_t n_kernels,
                         int32_t workers, int32_t fpk, double* out,
                         int64_t ld_out, int64_t row0);

/* The drop-in entry points with the arithmetic mode chosen by the caller
 * (RK_MODE_EXACT: byte-identical to the reference, as rk_run_batch_f32;
 * RK_MODE_FAST: the FFMA2 kernels within the north-star tolerance — the
 * headline kernels reached through the reference's own operator call).
 * Same arguments as rk_run_batch_f32 / _f64 plus mode; same return value.
 * float64 runs the reference loop in either mode (bytes equal). */
int64_t rk_run_batch_f32_mode(const float* x, int64_t n_instances,
                              int32_t n_channels, int32_t l_series,
                              const int32_t* lengths, const int32_t* dilations,
                              const int32_t* paddings, const float* biases,
                              const float* wflat, const int64_t* woff,
                              const int32_t* chidx, const int64_t* choff,
                              const int32_t* chcnt, int64_t n_kernels,
                              int32_t workers, int32_t fpk, float* out,
                              int64_t ld_out, int64_t row0, int32_t mode);
int64_t rk_run_batch_f64_mode(const double* x, int64_t n_instances,
                              int32_t n_channels, int32_t l_series,
                              const int32_t* lengths, const int32_t* dilations,
                              const int32_t* paddings, const double* biases,
                              const double* wflat, const int64_t* woff,
                              const int32_t* chidx, const int64_t* choff,
                              const int32_t* chcnt, int64_t n_kernels,
                              int32_t workers, int32_t fpk, double* out,
                              int64_t ld_out, int64_t row0, int32_t mode);

/* Streaming transform between files: the reference's
 * `gridrocket transform` reads the whole dataset (load_dataset,
 * data.py:293-302), transforms it in memory (cli.py:138-168) and saves the
 * FeatureMatrix (features.py:59-67).  This entry point does the same work
 * in bounded memory: n_series rows of n_channels*l_series values of type
 * in_dtype are read from in_fd at byte in_offset (or, when in_fd < 0, from
 * the host array x), converted to the compute dtype when they differ
 * (float64 -> float32 rounds to nearest, like numpy's astype), transformed,
 * and the (n_series, n_kernels*fpk) features of type dtype are written to
 * out_fd at byte out_offset — the bytes FeatureMatrix.save writes after its
 * header.  A reader thread (pread into pinned buffers), the GPU (H2D,
 * transform, D2H on separate streams) and a writer thread (pwrite from
 * pinned buffers) overlap batch by batch.  Non-finite inputs fail with
 * RK_ERR_INVALID, as engine._check_shapes does (engine.py:252-268), after
 * the rows before them were written.  batch_rows <= 0 picks a batch.
 * *executed (may be NULL) receives the positions counted on the device
 * (== positions_per_series * n_series). */
int rk_transform_stream(rk_bank_t bank, int32_t in_fd, int64_t in_offset,
                        const void* x, int32_t in_dtype, int64_t n_series,
                        int32_t out_fd, int64_t out_offset, int32_t dtype,
                        int32_t fpk, int32_t mode, int64_t batch_rows,
                        int64_t* executed);

/* Native bank generation: the reference's generate_bank
 * (kernels.py:243-308) — numpy Generator(Philox(key=seed)) draws in the
 * reference's per-kernel order (length, channel subset, weights, bias,
 * dilation, padding) — replayed bit for bit in C++ on the host (no GPU).
 * exponent_bounds[i] = float(np.log2((l_series-1)/(len_i-1))) for
 * len = 7, 9, 11 and channel_bound = float(np.log2(n_channels)), computed by
 * the caller with numpy as the reference does (kernels.py:204-214, 230-240).
 * Per-kernel outputs have count entries; channel_indices and weights are
 * filled up to index_capacity / weight_capacity (count*n_channels and
 * count*11*n_channels always suffice) and *n_indices / *n_weights receive
 * the lengths used.  Returns RK_ERR_CAPACITY if a buffer is too small — with
 * the lengths needed in *n_indices / *n_weights, so a caller can size its
 * buffers from an estimate and call again (the draw is deterministic). */
int rk_generate_bank(int64_t count, int32_t l_series, int32_t n_channels,
                     uint64_t seed, int32_t center_weights,
                     const double* exponent_bounds, double channel_bound,
                     int32_t* lengths, double* biases, int32_t* dilations,
                     int32_t* paddings, int32_t* channel_counts,
                     int32_t* channel_indices, int64_t index_capacity,
                     double* weights, int64_t weight_capacity,
                     int64_t* n_weights, int64_t* n_indices);

/* Release cached banks and per-device buffers (optional at exit). */
int rk_release_caches(void);

#ifdef __cplusplus
}
#endif
#endif /* ROCKET_B200_H */
