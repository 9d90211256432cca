"""Streaming file-to-file transform.

The reference's ``gridrocket transform`` (cli.py:138-168) loads the whole
dataset (data.py:293-302), transforms it in memory (engine.py:324-333) and
saves the FeatureMatrix (features.py:59-67).  ``transform_file`` produces
the same feature file byte for byte, but streams: the RKFM header is written
here and the native runtime (rk_transform_stream, csrc/rocket_stream.cu)
moves the rows disk -> pinned host buffers -> GPU -> pinned host buffers ->
disk with reads, copies, kernels and writes of consecutive batches
overlapped, so host memory stays bounded however large the dataset and the
feature matrix are.  A binary dataset cache (RKDS) is read straight from
the file; ``.ts`` / ``.csv`` inputs, and in-memory datasets, are parsed
first and streamed from memory.
"""

import ctypes
import os
import threading

import numpy as np

from . import _lib
from .data import Dataset, cache_layout, load_dataset
from .engine import (
    CapacityError,
    GridLimits,
    TransformStats,
    _check_request,
    bytes_per_instance,
    device_bank,
    plan_batches,
    plan_shards,
)
from .features import FEATURE_DATA_OFFSET, precision_dtype, write_feature_header
from .kernels import KernelBank


def _is_cache_path(path) -> bool:
    lower = str(path).lower()
    return not (lower.endswith(".ts") or lower.endswith(".csv"))


def _check_dims(n_channels, l_series, bank: KernelBank, limits: GridLimits):
    """The shape part of engine._check_shapes (engine.py:252-268); the
    finiteness scan runs natively while the rows stream."""
    if n_channels != bank.n_channels:
        raise ValueError(f"dataset has {n_channels} channels, bank was generated for {bank.n_channels}")
    if l_series != bank.l_series:
        raise ValueError(f"series length {l_series} does not match bank l_series {bank.l_series}")
    if bank.count > limits.max_x:
        raise CapacityError(f"{bank.count} kernels exceed the grid x-dimension limit {limits.max_x}")


def transform_file(
    data,
    bank: KernelBank,
    out_path,
    limits: GridLimits | None = None,
    include_mpv: bool = False,
    precision: str = "single",
    *,
    mode: str = "exact",
    device: int = 0,
    csv_labels: bool = False,
    batch_rows: int = 0,
    devices: int = 1,
) -> TransformStats:
    """Transform ``data`` (a dataset path — RKDS cache, ``.ts`` or ``.csv`` —
    a Dataset, or an (n, C, L) array) with ``bank`` and write the feature
    file ``out_path`` exactly as ``FeatureMatrix.save`` would.  On failure
    the partial output file is removed and the reference's exception type is
    raised (ValueError / CapacityError / FormatError / ParseError).

    ``devices`` > 1 splits the rows with plan_shards (engine.py:123-134)
    and streams every shard from its own host thread on its own GPU (round
    robin over the visible ones) into its own byte range of the one output
    file, as transform_sharded does in memory (engine.py:336-364)."""
    limits = GridLimits() if limits is None else limits
    _check_request(precision, mode)
    dtype = precision_dtype(precision)
    fpk = 3 if include_mpv else 2
    in_fd = -1
    values = None
    if isinstance(data, (str, os.PathLike)) and _is_cache_path(data):
        layout = cache_layout(data)
        n, n_channels, l_series = layout.n_instances, layout.n_channels, layout.l_series
        in_dtype = layout.dtype
        in_offset = layout.values_offset
    else:
        if isinstance(data, (str, os.PathLike)):
            data = load_dataset(data, csv_labels=csv_labels)
        values = np.asarray(data.values if isinstance(data, Dataset) else data)
        if values.ndim != 3:
            raise ValueError("expected values of shape (n_instances, n_channels, l_series)")
        if values.dtype not in (np.float32, np.float64):
            values = values.astype(np.float64)
        values = np.ascontiguousarray(values)
        n, n_channels, l_series = values.shape
        in_dtype = values.dtype.type
        in_offset = 0
    _check_dims(n_channels, l_series, bank, limits)
    # the reference's batch plan raises CapacityError when one series
    # exceeds the memory budget (engine.py:111-115), before any device work
    if n:
        plan_batches(n, bytes_per_instance(n_channels, l_series), limits)
    rk_dtype = _lib.RK_DTYPE_F64 if dtype == np.float64 else _lib.RK_DTYPE_F32
    in_rk = _lib.RK_DTYPE_F64 if in_dtype == np.float64 else _lib.RK_DTYPE_F32
    in_row = n_channels * l_series * np.dtype(in_dtype).itemsize
    out_row = bank.count * fpk * np.dtype(dtype).itemsize
    shards = [(s0, c) for s0, c in plan_shards(n, max(1, int(devices))) if c] if devices > 1 else [(0, n)]
    ngpu = max(1, _lib.device_count()) if len(shards) > 1 else 1
    stats = TransformStats(n_shards=len(shards))
    try:
        if values is None:
            in_fd = os.open(data, os.O_RDONLY)
        with open(out_path, "wb") as f:
            write_feature_header(f, n, bank.count, fpk, precision)
            f.flush()
            assert f.tell() == FEATURE_DATA_OFFSET
            executed = [0] * len(shards)
            errors = []

            def run(i, start, count):
                try:
                    dbank = device_bank(bank, (device + i) % ngpu if len(shards) > 1 else device)
                    if rk_dtype == _lib.RK_DTYPE_F64:
                        dbank.attach_f64()
                    ex = ctypes.c_int64(0)
                    x_ptr = values.ctypes.data + start * in_row if values is not None and count else None
                    rc = _lib.load().rk_transform_stream(
                        dbank.handle, in_fd, in_offset + start * in_row, ctypes.c_void_p(x_ptr), in_rk, count,
                        f.fileno(), FEATURE_DATA_OFFSET + start * out_row, rk_dtype, fpk, _lib.MODES[mode],
                        int(batch_rows), ctypes.byref(ex),
                    )
                    _lib.check(rc, "rk_transform_stream")
                    executed[i] = int(ex.value)
                except BaseException as e:  # re-raised on the caller thread
                    errors.append(e)

            if len(shards) == 1:
                run(0, *shards[0])
            else:
                threads = [threading.Thread(target=run, args=(i, s0, c)) for i, (s0, c) in enumerate(shards)]
                for t in threads:
                    t.start()
                for t in threads:
                    t.join()
            if errors:
                raise errors[0]
    except BaseException:
        if os.path.exists(out_path):
            os.remove(out_path)
        raise
    finally:
        if in_fd >= 0:
            os.close(in_fd)
    stats.total_dot_products = sum(executed)
    stats.n_batches = len(shards) if n else 0
    return stats
