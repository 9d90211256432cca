"""Transform engine: the reference's engine surface over the B200 kernels.

Mirrors /root/reference/pkg/src/gridrocket/engine.py — GridLimits,
plan_batches, plan_shards, CellAccumulator, transform, transform_with_stats,
transform_sharded — but the per-batch call that the reference makes into
numba (engine.py:280-295) goes through the C ABI (include/rocket_b200.h)
to hand-written sm_100a kernels.  There is no CPU fallback: without the
built library or a B200 the calls raise.

Arithmetic modes (keyword-only ``mode``):
  "exact" (default) — bit-identical to the reference engine (tap order,
                      bias last, no FMA contraction);
  "fast"            — FFMA2 with the bias folded in; within the north-star
                      tolerance (MAX 1e-5 relative, PPV exact except for
                      outputs within 1e-6 of zero).
precision="double" runs the cell kernels, which follow the reference loop
order exactly in both modes; include_mpv=True does too in "exact" mode
(the ordered positive sum, engine.py:193-249), while "fast" mode computes
MPV in the FFMA2 kernels from per-lane sums of the positive outputs (MPV
within 1e-5 relative, tests/parity.py).
"""

import ctypes
import hashlib
import os
import threading
from dataclasses import dataclass

import numpy as np

from . import _lib
from .features import FeatureMatrix, precision_dtype
from .kernels import KernelBank

SINGLE_BYTES = 4


class CapacityError(RuntimeError):
    """A work item cannot be scheduled within the configured limits
    (engine.py:30-31)."""


@dataclass
class GridLimits:
    """Grid-shape and memory constraints (engine.py:34-46).

    ``workers_per_cell`` is accepted for parity; as in the reference it
    cannot change any result.
    """

    max_x: int = 2**31 - 1
    max_y: int = 65535
    workers_per_cell: int = 1024
    memory_budget_bytes: int = 1 << 30

    def __post_init__(self):
        for name in ("max_x", "max_y", "workers_per_cell", "memory_budget_bytes"):
            if getattr(self, name) < 1:
                raise ValueError(f"{name} must be positive")


@dataclass
class EnginePlan:
    """Batch and shard schedule of one transform (engine.py:49-55)."""

    batches: list
    shards: list
    bytes_per_instance: int


@dataclass
class CellAccumulator:
    """Reduction state of one (series, kernel) cell (engine.py:58-79).

    (count, +) and (max, -inf) are commutative monoids; the CUDA epilogue
    reduces per-lane states with the same monoids (warp REDUX add / max).
    """

    ppv_count: int = 0
    running_max: float = float("-inf")

    def update(self, is_positive: bool, dot_value: float) -> None:
        if is_positive:
            self.ppv_count += 1
        if dot_value > self.running_max:
            self.running_max = dot_value

    def merge(self, other: "CellAccumulator") -> "CellAccumulator":
        return CellAccumulator(
            ppv_count=self.ppv_count + other.ppv_count,
            running_max=max(self.running_max, other.running_max),
        )


@dataclass
class TransformStats:
    """Execution accounting (engine.py:82-88).  total_dot_products is
    counted on the device by the kernels."""

    total_dot_products: int = 0
    n_batches: int = 0
    n_shards: int = 1


def reduce_cell(updates) -> CellAccumulator:
    """Fold (is_positive, value) updates (engine.py:91-96)."""
    acc = CellAccumulator()
    for is_positive, dot_value in updates:
        acc.update(is_positive, dot_value)
    return acc


def bytes_per_instance(n_channels: int, l_series: int) -> int:
    """Planning size of one series (engine.py:99-101)."""
    return int(n_channels) * int(l_series) * SINGLE_BYTES


def plan_batches(n_instances: int, bytes_per_instance: int, limits: GridLimits) -> EnginePlan:
    """Ordered row batches under the y-limit and memory budget
    (engine.py:104-120)."""
    if n_instances < 0:
        raise ValueError("n_instances must be non-negative")
    if bytes_per_instance < 1:
        raise ValueError("bytes_per_instance must be positive")
    fits = limits.memory_budget_bytes // bytes_per_instance
    if fits < 1:
        raise CapacityError(
            f"one instance needs {bytes_per_instance} bytes but the budget is "
            f"{limits.memory_budget_bytes}"
        )
    size = min(limits.max_y, int(fits))
    batches = [(s, min(size, n_instances - s)) for s in range(0, n_instances, size)]
    return EnginePlan(batches=batches, shards=[(0, n_instances)], bytes_per_instance=bytes_per_instance)


def plan_shards(n_instances: int, n_devices: int) -> list:
    """n_devices contiguous near-equal row ranges (engine.py:123-134)."""
    if n_devices < 1:
        raise ValueError("n_devices must be positive")
    base, extra = divmod(n_instances, n_devices)
    shards, start = [], 0
    for d in range(n_devices):
        size = base + (1 if d < extra else 0)
        shards.append((start, size))
        start += size
    return shards


def total_positions(bank: KernelBank) -> int:
    """Sum of l_out over the bank (engine.py:137-141)."""
    return int(bank.output_lengths().sum())


def expected_dot_products(bank: KernelBank, n_instances: int) -> int:
    return total_positions(bank) * int(n_instances)


def useful_flops_per_series(bank: KernelBank) -> int:
    """Algorithmic FLOPs of one series: sum_k 2*(in-range taps) + l_out
     — the roofline numerator."""
    lk = bank.lengths.astype(np.int64)
    d = bank.dilations.astype(np.int64)
    p = bank.paddings.astype(np.int64)
    nc = bank.channel_counts.astype(np.int64)
    l_out = bank.output_lengths()
    taps = np.zeros(bank.count, dtype=np.int64)
    for j in range(int(lk.max())):
        live = j < lk
        off = j * d - p
        lo = np.maximum(0, -off)
        hi = np.minimum(l_out, bank.l_series - off)
        taps += np.where(live, np.maximum(hi - lo, 0), 0)
    return int((2 * taps * nc + l_out).sum())


_finite_pool = None


def _all_finite(values: np.ndarray) -> bool:
    """np.isfinite(values).all(), split over host threads for large inputs
    (numpy releases the GIL in the scan; config 2's 410 MB took 57 ms on one
    core of the GPU box)."""
    global _finite_pool
    v = np.asarray(values)
    threads = min(16, len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1))
    if v.size < (1 << 23) or v.ndim == 0 or v.shape[0] < 2 * threads or threads < 2:
        return bool(np.isfinite(v).all())
    if _finite_pool is None:
        from concurrent.futures import ThreadPoolExecutor

        _finite_pool = ThreadPoolExecutor(max_workers=threads)
    bounds = np.linspace(0, v.shape[0], threads + 1).astype(int)
    parts = [v[a:b] for a, b in zip(bounds[:-1], bounds[1:])]
    return all(_finite_pool.map(lambda p: bool(np.isfinite(p).all()), parts))


def _check_shapes(values: np.ndarray, bank: KernelBank, limits: GridLimits) -> None:
    """engine.py:252-268."""
    if values.ndim != 3:
        raise ValueError("expected values of shape (n_instances, n_channels, l_series)")
    if values.shape[1] != bank.n_channels:
        raise ValueError(
            f"dataset has {values.shape[1]} channels, bank was generated for {bank.n_channels}"
        )
    if values.shape[2] != bank.l_series:
        raise ValueError(
            f"series length {values.shape[2]} does not match bank l_series {bank.l_series}"
        )
    if bank.count > limits.max_x:
        raise CapacityError(f"{bank.count} kernels exceed the grid x-dimension limit {limits.max_x}")
    if not _all_finite(values):
        raise ValueError("dataset contains non-finite values")


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def bank_identity(bank: KernelBank) -> str:
    """Content hash of everything the device layout depends on."""
    h = hashlib.sha1()
    h.update(np.array([bank.count, bank.l_series, bank.n_channels], dtype=np.int64).tobytes())
    for arr in (
        bank.lengths,
        bank.dilations,
        bank.paddings,
        bank.channel_counts,
        bank.channel_indices,
        bank.weights,
        bank.biases,
    ):
        h.update(np.ascontiguousarray(arr).tobytes())
    return h.hexdigest()


class DeviceBank:
    """A KernelBank laid out on one GPU (rk_bank_create): kernels grouped by
    (length, dilation, padding, channel set) into warp chunks."""

    def __init__(self, bank: KernelBank, device: int = 0):
        lib = _lib.load()
        self.bank = bank
        self.device = int(device)
        self._keep = dict(
            lengths=np.ascontiguousarray(bank.lengths, dtype=np.int32),
            dilations=np.ascontiguousarray(bank.dilations, dtype=np.int32),
            paddings=np.ascontiguousarray(bank.paddings, dtype=np.int32),
            # f64 bank -> f32 round-to-nearest once, as engine._run_range (engine.py:275-276)
            biases=np.ascontiguousarray(bank.biases.astype(np.float32)),
            weights=np.ascontiguousarray(bank.weights.astype(np.float32)),
            woff=np.ascontiguousarray(bank.weight_offsets, dtype=np.int64),
            chidx=np.ascontiguousarray(bank.channel_indices, dtype=np.int32),
            choff=np.ascontiguousarray(bank.channel_offsets, dtype=np.int64),
            chcnt=np.ascontiguousarray(bank.channel_counts, dtype=np.int32),
        )
        k = self._keep
        handle = ctypes.c_void_p()
        rc = lib.rk_bank_create(
            bank.count, bank.n_channels, bank.l_series,
            _ptr(k["lengths"]), _ptr(k["dilations"]), _ptr(k["paddings"]), _ptr(k["biases"]),
            _ptr(k["weights"]), _ptr(k["woff"]), _ptr(k["chidx"]), _ptr(k["choff"]), _ptr(k["chcnt"]),
            self.device, ctypes.byref(handle),
        )
        _lib.check(rc, "rk_bank_create")
        self._handle = handle
        self._f64 = False
        self._f64_lock = threading.Lock()
        info = _lib.BankInfo()
        _lib.check(lib.rk_bank_info(handle, ctypes.byref(info)), "rk_bank_info")
        self.info = {f: getattr(info, f) for f, _ in _lib.BankInfo._fields_}

    @property
    def handle(self):
        return self._handle

    def attach_f64(self):
        """Upload the float64 bank parameters (precision "double"); shard
        threads sharing this bank attach it once, and none transforms before
        the upload is complete."""
        with self._f64_lock:
            if self._f64:
                return
            bank = self.bank
            self._keep["biases64"] = np.ascontiguousarray(bank.biases, dtype=np.float64)
            self._keep["weights64"] = np.ascontiguousarray(bank.weights, dtype=np.float64)
            rc = _lib.load().rk_bank_attach_f64(self._handle, _ptr(self._keep["biases64"]),
                                                _ptr(self._keep["weights64"]))
            _lib.check(rc, "rk_bank_attach_f64")
            self._f64 = True

    def transform_into(self, x_ptr, n_series, out_ptr, ld_out, row0=0, mode="exact", stream=None, fpk=2,
                       precision="single"):
        """Raw-pointer transform (host or device pointers); returns the
        device-counted executed positions."""
        lib = _lib.load()
        dtype = _lib.RK_DTYPE_F64 if precision == "double" else _lib.RK_DTYPE_F32
        if dtype == _lib.RK_DTYPE_F64:
            self.attach_f64()
        executed = ctypes.c_int64(0)
        rc = lib.rk_transform(
            self._handle, ctypes.c_void_p(x_ptr), dtype, int(n_series), ctypes.c_void_p(out_ptr), int(ld_out),
            int(row0), int(fpk), _lib.MODES[mode], ctypes.c_void_p(stream or 0), ctypes.byref(executed),
        )
        _lib.check(rc, "rk_transform")
        return int(executed.value)

    def close(self):
        if getattr(self, "_handle", None):
            try:
                _lib.load().rk_bank_destroy(self._handle)
            finally:
                self._handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_bank_cache = {}
_bank_lock = threading.Lock()


def device_bank(bank: KernelBank, device: int = 0) -> DeviceBank:
    """Cached DeviceBank keyed by bank content and device."""
    key = (bank_identity(bank), int(device))
    with _bank_lock:
        db = _bank_cache.get(key)
        if db is None:
            if len(_bank_cache) >= 8:
                # dropped, not closed: a thread may still be transforming
                # with it; __del__ frees it once the last user lets go
                _bank_cache.pop(next(iter(_bank_cache)))
            db = DeviceBank(bank, device)
            _bank_cache[key] = db
        return db


def _check_request(precision, mode):
    precision_dtype(precision)
    if mode not in _lib.MODES:
        raise ValueError(f"mode must be one of {sorted(_lib.MODES)}")


def _run_range(x, dbank, limits, out, row0, stats, mode, fpk, precision):
    """engine.py:271-296.  The reference's batch plan (and its CapacityError)
    is kept and reported in stats.n_batches, but the rows go to the library
    in one call: its pinned-ring pipeline already bounds host and device
    memory, and one pipeline instead of one per planned batch saves a fill
    and drain per batch (rows are independent, so the features are the same
    bytes — test_sharding_and_batching_are_pure_partitions)."""
    plan = plan_batches(x.shape[0], bytes_per_instance(x.shape[1], x.shape[2]), limits)
    if x.shape[0]:
        stats.total_dot_products += dbank.transform_into(
            x.ctypes.data, x.shape[0], out.ctypes.data, out.shape[1], row0, mode=mode, fpk=fpk, precision=precision,
        )
    stats.n_batches += len(plan.batches)


def transform_with_stats(
    data,
    bank: KernelBank,
    limits: GridLimits | None = None,
    include_mpv: bool = False,
    precision: str = "single",
    *,
    mode: str = "exact",
    device: int = 0,
):
    """Like :func:`transform` but also returns TransformStats
    (engine.py:299-321)."""
    limits = GridLimits() if limits is None else limits
    values = np.asarray(getattr(data, "values", data))
    _check_shapes(values, bank, limits)
    _check_request(precision, mode)
    dtype = precision_dtype(precision)
    fpk = 3 if include_mpv else 2
    x = np.ascontiguousarray(values, dtype=dtype)
    out = np.empty((values.shape[0], bank.count * fpk), dtype=dtype)
    stats = TransformStats()
    if values.shape[0]:
        _run_range(x, device_bank(bank, device), limits, out, 0, stats, mode, fpk, precision)
    matrix = FeatureMatrix(values=out, n_kernels=bank.count, features_per_kernel=fpk, precision=precision)
    return matrix, stats


def transform(
    data,
    bank: KernelBank,
    limits: GridLimits | None = None,
    include_mpv: bool = False,
    precision: str = "single",
    *,
    mode: str = "exact",
    device: int = 0,
) -> FeatureMatrix:
    """Transform every series with every kernel on the GPU (engine.py:324-333)."""
    matrix, _ = transform_with_stats(data, bank, limits, include_mpv, precision, mode=mode, device=device)
    return matrix


def transform_sharded(
    data,
    bank: KernelBank,
    n_devices: int,
    limits: GridLimits | None = None,
    include_mpv: bool = False,
    precision: str = "single",
    *,
    mode: str = "exact",
    devices=None,
) -> FeatureMatrix:
    """Split series into n_devices contiguous shards (plan_shards), run each
    shard on its own GPU from its own host thread, and write the row blocks
    in place (engine.py:336-364).  With fewer visible GPUs than shards the
    shards are assigned round-robin; the result is identical for any split."""
    limits = GridLimits() if limits is None else limits
    values = np.asarray(getattr(data, "values", data))
    _check_shapes(values, bank, limits)
    _check_request(precision, mode)
    dtype = precision_dtype(precision)
    fpk = 3 if include_mpv else 2
    x = np.ascontiguousarray(values, dtype=dtype)
    out = np.empty((values.shape[0], bank.count * fpk), dtype=dtype)
    shards = [(s, c) for s, c in plan_shards(values.shape[0], n_devices) if c]
    if shards:
        if devices is None:
            ngpu = max(1, _lib.device_count())
            devices = [i % ngpu for i in range(len(shards))]
        errors = []

        def run(shard, dev):
            start, count = shard
            try:
                st = TransformStats()
                _run_range(x[start : start + count], device_bank(bank, dev), limits, out, start, st, mode, fpk,
                           precision)
            except BaseException as e:  # re-raised on the caller thread
                errors.append(e)

        threads = [threading.Thread(target=run, args=(s, devices[i])) for i, s in enumerate(shards)]
        for t in threads:
            t.start()
        for t in threads:
            t.join()
        if errors:
            raise errors[0]
    return FeatureMatrix(values=out, n_kernels=bank.count, features_per_kernel=fpk, precision=precision)
