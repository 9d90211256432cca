"""GPU parity: the CUDA transform (through the C ABI) vs the reference.

Exact mode must be byte-identical to the reference's single-precision
engine (golden fixtures from gridrocket.transform, and the pinned oracle);
fast mode must meet the north-star tolerance (tests/parity.py)."""

import ctypes

import numpy as np
import pytest

import golden_cases as gc
from parity import check_fast
from paper_2601_17091_b200 import (
    CapacityError,
    GenOptions,
    GridLimits,
    device_bank,
    expected_dot_products,
    generate_bank,
    synth_random,
    transform,
    transform_sharded,
    transform_with_stats,
)

pytestmark = pytest.mark.gpu
SINGLE = [name for name, case in gc.CASES.items() if "single" in case["variants"]]


def _case(name):
    case = gc.CASES[name]
    return gc.case_values(case), gc.make_bank(gc.BANKS[case["bank"]])


@pytest.mark.parametrize("name", SINGLE)
def test_exact_bytes_match_reference(name, golden_transforms, cuda_ready):
    values, bank = _case(name)
    fm, stats = transform_with_stats(values, bank, mode="exact")
    ref = golden_transforms[f"{name}/single"]
    assert fm.values.dtype == np.float32 and fm.values.shape == ref.shape
    assert fm.values.tobytes() == ref.tobytes()
    assert stats.total_dot_products == int(golden_transforms[f"{name}/single/executed"][0])


@pytest.mark.parametrize("name", SINGLE)
def test_fast_within_tolerance(name, golden_transforms, cuda_ready):
    values, bank = _case(name)
    fm = transform(values, bank, mode="fast")
    check_fast(fm.values, golden_transforms[f"{name}/single"], values, bank)


def test_run_batch_dropin_signature(golden_transforms, cuda_ready):
    """rk_run_batch_f32 takes _run_batch's argument list (engine.py:148-150)."""
    lib = cuda_ready
    values, bank = _case("rc7")
    x = np.ascontiguousarray(values, dtype=np.float32)
    out = np.full((x.shape[0] + 3, bank.count * 2), np.nan, dtype=np.float32)
    a = dict(
        lengths=bank.lengths, dilations=bank.dilations, paddings=bank.paddings,
        biases=bank.biases.astype(np.float32), wflat=bank.weights.astype(np.float32),
        woff=bank.weight_offsets, chidx=bank.channel_indices, choff=bank.channel_offsets,
        chcnt=bank.channel_counts,
    )
    a = {k: np.ascontiguousarray(v) for k, v in a.items()}
    p = lambda arr: arr.ctypes.data_as(ctypes.c_void_p)  # noqa: E731
    executed = lib.rk_run_batch_f32(
        p(x), x.shape[0], x.shape[1], x.shape[2], p(a["lengths"]), p(a["dilations"]), p(a["paddings"]),
        p(a["biases"]), p(a["wflat"]), p(a["woff"]), p(a["chidx"]), p(a["choff"]), p(a["chcnt"]),
        bank.count, 1024, 2, p(out), out.shape[1], 3,
    )
    assert executed == expected_dot_products(bank, x.shape[0])
    assert np.isnan(out[:3]).all()
    assert out[3:].tobytes() == golden_transforms["rc7/single"].tobytes()


def test_run_batch_mpv_dropin(golden_transforms, cuda_ready):
    """fpk = 3 through rk_run_batch_f32: _run_batch_mpv's bytes."""
    lib = cuda_ready
    values, bank = _case("small")
    x = np.ascontiguousarray(values, dtype=np.float32)
    out = np.empty((x.shape[0], bank.count * 3), dtype=np.float32)
    arrs = [np.ascontiguousarray(v) for v in (
        bank.lengths, bank.dilations, bank.paddings, bank.biases.astype(np.float32),
        bank.weights.astype(np.float32), bank.weight_offsets, bank.channel_indices, bank.channel_offsets,
        bank.channel_counts)]
    p = lambda arr: arr.ctypes.data_as(ctypes.c_void_p)  # noqa: E731
    executed = lib.rk_run_batch_f32(p(x), x.shape[0], x.shape[1], x.shape[2], *[p(a) for a in arrs],
                                    bank.count, 1024, 3, p(out), out.shape[1], 0)
    assert executed == expected_dot_products(bank, x.shape[0])
    assert out.tobytes() == golden_transforms["small/single_mpv"].tobytes()


def test_sharding_and_batching_are_pure_partitions(cuda_ready):
    values, bank = _case("rc300")
    whole = transform(values, bank)
    assert transform_sharded(values, bank, 4).values.tobytes() == whole.values.tobytes()
    fm, stats = transform_with_stats(values, bank, limits=GridLimits(max_y=7, workers_per_cell=3))
    assert fm.values.tobytes() == whole.values.tobytes()
    assert stats.n_batches == -(-values.shape[0] // 7)
    assert stats.total_dot_products == expected_dot_products(bank, values.shape[0])
    empty = transform_sharded(np.zeros((0, 1, bank.l_series)), bank, 3)
    assert empty.values.shape == (0, bank.count * 2)


def test_fast_mode_is_deterministic(cuda_ready):
    values, bank = _case("l1024")
    a = transform(values, bank, mode="fast").values
    b = transform(values, bank, mode="fast").values
    assert a.tobytes() == b.tobytes()


def test_device_pointer_path_matches_host_path(golden_transforms, cuda_ready):
    import torch

    values, bank = _case("mv2048")
    db = device_bank(bank, 0)
    x = torch.from_numpy(np.ascontiguousarray(values, dtype=np.float32)).cuda()
    out = torch.full((x.shape[0] + 1, bank.count * 2), float("nan"), device="cuda")
    stream = torch.cuda.current_stream().cuda_stream
    executed = db.transform_into(x.data_ptr(), x.shape[0], out.data_ptr(), out.shape[1], row0=1,
                                 mode="exact", stream=stream)
    torch.cuda.synchronize()
    assert executed == expected_dot_products(bank, x.shape[0])
    got = out.cpu().numpy()
    assert np.isnan(got[0]).all()
    assert got[1:].tobytes() == golden_transforms["mv2048/single"].tobytes()


def test_config2_rows_exact_vs_oracle(cuda_ready):
    """BASELINE config 2 shape (L=1024, 10k kernels) on a 192-series slice."""
    from oracle.oracle import oracle_transform

    bank = generate_bank(1024, 1, 10000, GenOptions(seed=0))
    values = synth_random(192, 1, 1024, seed=1).values
    got = transform(values, bank, mode="exact").values
    assert got.tobytes() == oracle_transform(values, bank).tobytes()


def test_config5_multichannel_exact_vs_oracle(cuda_ready):
    """BASELINE config 5 shape (3 channels, L=2048) at 10k kernels, 24 series."""
    from oracle.oracle import oracle_transform

    bank = generate_bank(2048, 3, 10000, GenOptions(seed=0))
    values = synth_random(24, 3, 2048, seed=1).values
    got = transform(values, bank, mode="exact").values
    assert got.tobytes() == oracle_transform(values, bank).tobytes()
    fast = transform(values, bank, mode="fast").values
    check_fast(fast, got, values, bank)


def test_full_size_config2_properties(cuda_ready):
    """Full BASELINE config 2 (100k x 1024, 10k kernels) device-resident:
    size-independent properties + sampled rows vs the oracle."""
    import torch

    from oracle.oracle import oracle_transform

    bank = generate_bank(1024, 1, 10000, GenOptions(seed=0))
    n = 100_000
    g = torch.Generator(device="cuda").manual_seed(1)
    x = torch.randn((n, 1, 1024), device="cuda", generator=g, dtype=torch.float32)
    out = torch.empty((n, bank.count * 2), device="cuda", dtype=torch.float32)
    db = device_bank(bank, 0)
    executed = db.transform_into(x.data_ptr(), n, out.data_ptr(), out.shape[1], mode="exact",
                                 stream=torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    assert executed == expected_dot_products(bank, n)
    ppv = out[:, 0::2]
    l_out = torch.from_numpy(bank.output_lengths()).cuda().to(torch.float64)
    counts = ppv.to(torch.float64) * l_out
    assert torch.all((counts - counts.round()).abs() < 1e-3)
    assert torch.all((ppv >= 0) & (ppv <= 1))
    rows = torch.tensor([0, 1, 4242, 50_000, 77_777, n - 1], device="cuda")
    sample = x[rows].cpu().numpy()
    assert out[rows].cpu().numpy().tobytes() == oracle_transform(sample, bank).tobytes()


def test_errors_mirror_reference(cuda_ready):
    values, bank = _case("small")
    with pytest.raises(ValueError):
        transform(np.zeros((2, 2, 64)), bank)
    with pytest.raises(ValueError):
        transform(np.zeros((2, 1, 32)), bank)
    bad = np.zeros((2, 1, 64))
    bad[1, 0, 5] = np.inf
    with pytest.raises(ValueError):
        transform(bad, bank)
    with pytest.raises(CapacityError):
        transform(values, bank, limits=GridLimits(max_x=3))
    with pytest.raises(ValueError):
        transform(values, bank, mode="approximate")
    # a series longer than shared memory holds is no longer a capacity
    # error: the GMEM kernels read it from global memory (test_gpu_long.py)
    big = generate_bank(200_000, 1, 4, GenOptions(seed=3))
    assert transform(np.zeros((1, 1, 200_000), dtype=np.float32), big).values.shape == (1, 8)


OTHER = [(name, v) for name, case in gc.CASES.items() for v in case["variants"] if v != "single"]


@pytest.mark.parametrize("name,variant", OTHER)
def test_double_and_mpv_bytes_match_reference(name, variant, golden_transforms, cuda_ready):
    """precision="double" (both modes) and include_mpv=True in exact mode run
    the cell kernels: bytes equal.  Single-precision MPV in fast mode runs
    the wide kernels: the fast tolerance, MPV included."""
    values, bank = _case(name)
    precision = variant.split("_")[0]
    mpv = variant.endswith("_mpv")
    ref = golden_transforms[f"{name}/{variant}"]
    for mode in ("exact", "fast"):
        fm, stats = transform_with_stats(values, bank, include_mpv=mpv, precision=precision, mode=mode)
        assert fm.values.dtype == ref.dtype and fm.values.shape == ref.shape
        if mode == "fast" and mpv and precision == "single":
            check_fast(fm.values, ref, values, bank, fpk=3)
        else:
            assert fm.values.tobytes() == ref.tobytes()
        assert stats.total_dot_products == int(golden_transforms[f"{name}/{variant}/executed"][0])


def test_fast_mpv_config2_rows(cuda_ready):
    """Fast-mode MPV (wide kernels) at the BASELINE shape: PPV/MAX within the
    north-star tolerance, MPV within 1e-5 relative (certified cells aside)."""
    from oracle.oracle import oracle_transform

    bank = generate_bank(1024, 1, 10000, GenOptions(seed=0))
    values = synth_random(16, 1, 1024, seed=1).values
    ref = oracle_transform(values, bank, include_mpv=True)
    rep = check_fast(transform(values, bank, include_mpv=True, mode="fast").values, ref, values, bank, fpk=3)
    assert rep["cells"] == 16 * 10000


def test_mpv_and_double_config2_rows_vs_oracle(cuda_ready):
    """MPV (single) and double precision at the BASELINE L=1024 / 10k shape."""
    from oracle.oracle import oracle_transform

    bank = generate_bank(1024, 1, 10000, GenOptions(seed=0))
    values = synth_random(8, 1, 1024, seed=1).values
    mpv = transform(values, bank, include_mpv=True).values
    assert mpv.tobytes() == oracle_transform(values, bank, include_mpv=True).tobytes()
    dbl = transform(values, bank, precision="double").values
    assert dbl.tobytes() == oracle_transform(values, bank, precision="double").tobytes()


def test_staged_and_unstaged_cell_kernels_agree(cuda_ready, monkeypatch):
    """The staged cell kernel (series in shared memory) and the unstaged one
    (its fallback when a series does not fit) are both the reference's loop:
    identical bytes, multichannel MPV and double."""
    bank = generate_bank(96, 5, 300, GenOptions(seed=21))
    values = synth_random(40, 5, 96, seed=22).values
    staged = [transform(values, bank, include_mpv=True).values,
              transform(values, bank, precision="double", include_mpv=True).values]
    monkeypatch.setenv("RK_NO_CELLROW", "1")
    unstaged = [transform(values, bank, include_mpv=True).values,
                transform(values, bank, precision="double", include_mpv=True).values]
    for a, b in zip(staged, unstaged):
        assert a.tobytes() == b.tobytes()


def test_double_long_series_vs_oracle(cuda_ready):
    """L = 16384 in float64 needs more shared memory than an SM has for one
    staged series: the unstaged cell kernel runs, still byte-identical."""
    from oracle.oracle import oracle_transform

    bank = generate_bank(16384, 1, 120, GenOptions(seed=0))
    values = synth_random(2, 1, 16384, seed=1).values
    out = transform(values, bank, precision="double", include_mpv=True).values
    assert out.tobytes() == oracle_transform(values, bank, precision="double", include_mpv=True).tobytes()


def test_run_batch_f64_dropin(golden_transforms, cuda_ready):
    lib = cuda_ready
    values, bank = _case("rc5")
    x = np.ascontiguousarray(values, dtype=np.float64)
    out = np.empty((x.shape[0], bank.count * 2), dtype=np.float64)
    a = dict(
        lengths=bank.lengths, dilations=bank.dilations, paddings=bank.paddings, biases=bank.biases,
        wflat=bank.weights, woff=bank.weight_offsets, chidx=bank.channel_indices, choff=bank.channel_offsets,
        chcnt=bank.channel_counts,
    )
    a = {k: np.ascontiguousarray(v) for k, v in a.items()}
    p = lambda arr: arr.ctypes.data_as(ctypes.c_void_p)  # noqa: E731
    executed = lib.rk_run_batch_f64(
        p(x), x.shape[0], x.shape[1], x.shape[2], p(a["lengths"]), p(a["dilations"]), p(a["paddings"]),
        p(a["biases"]), p(a["wflat"]), p(a["woff"]), p(a["chidx"]), p(a["choff"]), p(a["chcnt"]),
        bank.count, 7, 2, p(out), out.shape[1], 0,
    )
    assert executed == expected_dot_products(bank, x.shape[0])
    assert out.tobytes() == golden_transforms["rc5/double"].tobytes()


def test_class_kernel_path_still_exact(cuda_ready, monkeypatch):
    """RK_NO_WIDE_PATH (read when the device bank is built) runs every chunk
    on the class kernel, including the 1-position generic path for 3+
    channel slots: same bytes as the oracle."""
    from oracle.oracle import oracle_transform

    monkeypatch.setenv("RK_NO_WIDE_PATH", "1")
    bank = generate_bank(96, 6, 150, GenOptions(seed=4242))
    values = synth_random(11, 6, 96, seed=4243).values
    out = transform(values, bank).values
    assert out.tobytes() == oracle_transform(values, bank).tobytes()


def test_concurrent_callers_on_one_stream(cuda_ready):
    """Several host threads transforming device buffers on the library's
    default stream (stream=None) at once: each call's counter reset, launch
    chain and executed-count read stay together (SPEC.md:267 — safe from
    concurrent callers on distinct outputs)."""
    import threading

    import torch

    bank = generate_bank(256, 1, 600, GenOptions(seed=31))
    db = device_bank(bank, 0)
    xs = [torch.from_numpy(synth_random(300 + 17 * i, 1, 256, seed=40 + i).values).cuda() for i in range(6)]
    ref = [transform(x.cpu().numpy(), bank).values for x in xs]
    outs = [torch.empty((x.shape[0], bank.count * 2), device="cuda") for x in xs]
    executed = [0] * len(xs)
    errors = []

    def run(i):
        try:
            for _ in range(3):
                executed[i] = db.transform_into(xs[i].data_ptr(), xs[i].shape[0], outs[i].data_ptr(),
                                                bank.count * 2, mode="exact")
        except BaseException as e:  # pragma: no cover - reported below
            errors.append(e)

    threads = [threading.Thread(target=run, args=(i,)) for i in range(len(xs))]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert not errors
    torch.cuda.synchronize()
    for i, x in enumerate(xs):
        assert outs[i].cpu().numpy().tobytes() == ref[i].tobytes()
        assert executed[i] == expected_dot_products(bank, x.shape[0])


@pytest.mark.parametrize("n", [3601, 9000])
def test_half_warp_chunks_exact(n, cuda_ready):
    """Enough series for two-series items, so the single-channel chunks run
    as half-warp chunks (16 lanes per series; an odd last series shadowed by
    the upper half): bytes equal to the oracle on every row, fast mode (with
    and without MPV) within tolerance."""
    from oracle.oracle import oracle_transform

    bank = generate_bank(256, 1, 300, GenOptions(seed=77))
    values = synth_random(n, 1, 256, seed=78).values
    ref = oracle_transform(values, bank)
    assert transform(values, bank, mode="exact").values.tobytes() == ref.tobytes()
    check_fast(transform(values, bank, mode="fast").values, ref, values, bank)
    ref3 = oracle_transform(values, bank, include_mpv=True)
    check_fast(transform(values, bank, include_mpv=True, mode="fast").values, ref3, values, bank, fpk=3)


@pytest.mark.parametrize("channels", [1, 3])
def test_position_paired_chunks(channels, cuda_ready, monkeypatch):
    """Lone kernels (a group of one) run position-paired: the two FFMA2 lanes
    hold two positions of the one kernel (kinds 6 / 7, 1 or 2 channel
    slots).  Exact mode stays byte-identical to the oracle and to the layout
    without pairing (RK_NO_SP); fast mode (with MPV) within tolerance."""
    from oracle.oracle import oracle_transform

    bank = generate_bank(2048, channels, 400, GenOptions(seed=91))
    db = device_bank(bank, 0)
    assert db.info["n_paired_chunks"] > 0
    values = synth_random(700, channels, 2048, seed=92).values
    ref = oracle_transform(values[:40], bank)
    exact = transform(values, bank, mode="exact").values
    assert exact[:40].tobytes() == ref.tobytes()
    check_fast(transform(values[:40], bank, mode="fast").values, ref, values[:40], bank)
    ref3 = oracle_transform(values[:40], bank, include_mpv=True)
    check_fast(transform(values[:40], bank, mode="fast", include_mpv=True).values, ref3, values[:40], bank, fpk=3)
    monkeypatch.setenv("RK_NO_SP", "1")
    from paper_2601_17091_b200.engine import DeviceBank

    plain = DeviceBank(bank, 0)
    assert plain.info["n_paired_chunks"] == 0
    import torch

    x = torch.from_numpy(values).cuda()
    out = torch.empty((values.shape[0], bank.count * 2), device="cuda")
    plain.transform_into(x.data_ptr(), values.shape[0], out.data_ptr(), out.shape[1], mode="exact")
    torch.cuda.synchronize()
    assert out.cpu().numpy().tobytes() == exact.tobytes()
    plain.close()
