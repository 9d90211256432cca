"""Parity on exactly the paths bench.py times.

* Device-resident fast mode at the BASELINE sizes (config 2: 100,000 x
  1,024; config 4: 20,000 x 16,384; config 5: 50,000 x 3 x 2,048; the
  FordA shape and 50,000 x 2,048 the bench also reports): enough series
  that items stage two or more series and the single-channel chunks run as
  half-warp chunks, as in the timed region.  Sampled rows are compared with
  the oracle under the north-star tolerance (oracle/parity.py: MAX within
  1e-5 relative, PPV flips only at float32-undecided outputs, both
  certified against float64), exact mode byte for byte on the same rows,
  and the device-counted executed positions with expected_dot_products
  (engine.py:137-145).
* The pinned-host pipeline bench.py's e2e calls (rk_transform with pinned
  x / out: row batches through a pooled worker on three streams) and the
  pageable numpy path of the public transform(): bytes equal to the
  device-pointer path in both modes, fpk 2 and 3, float32 and float64.

Reference: /root/reference/pkg/src/gridrocket/engine.py:148-190 (the
per-cell loop), SPEC.md:450-459 (acceptance criteria)."""

import os

import numpy as np
import pytest

from parity import check_fast
from paper_2601_17091_b200 import GenOptions, device_bank, expected_dot_products, generate_bank, synth_random

pytestmark = pytest.mark.gpu

# (name, n, C, L, row stride of the oracle sample)
BENCHED = [
    ("config2", 100_000, 1, 1024, 50),
    ("config4", 20_000, 1, 16_384, 100),
    ("config5", 50_000, 3, 2048, 100),
    ("forda", 3_601, 1, 500, 1),
    ("uni2048", 50_000, 1, 2048, 100),
]


def _device_transform(db, x_dev, n, fpk, mode, precision="single"):
    import torch

    dt = torch.float64 if precision == "double" else torch.float32
    out = torch.empty((n, db.bank.count * fpk), device="cuda", dtype=dt)
    executed = db.transform_into(x_dev.data_ptr(), n, out.data_ptr(), out.shape[1], mode=mode, fpk=fpk,
                                 precision=precision, stream=torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    return out, executed


@pytest.mark.parametrize("name,n,c,l,stride", BENCHED, ids=[b[0] for b in BENCHED])
def test_benched_fast_path_full_size(name, n, c, l, stride, cuda_ready):
    import torch

    from oracle.oracle import oracle_transform

    bank = generate_bank(l, c, 10_000, GenOptions(seed=0))
    values = synth_random(n, c, l, seed=1).values  # bench.py's inputs
    db = device_bank(bank, 0)
    if c == 1 and l <= 2048:
        # the layout the bench runs: half-warp chunks (two series per pass)
        assert db.info["n_half_chunks"] + db.info["n_quarter_chunks"] + db.info["n_eighth_chunks"] > 0
    assert db.info["n_runmajor_chunks"] > 0  # both lane-map orders run in the timed layout
    x = torch.from_numpy(values).cuda()
    rows = np.arange(0, n, stride)
    rows[-1] = n - 1
    sample = values[rows]
    ref = oracle_transform(sample, bank)
    fast, executed = _device_transform(db, x, n, 2, "fast")
    assert executed == expected_dot_products(bank, n)
    got = fast[torch.from_numpy(rows).cuda()].cpu().numpy()
    del fast
    rep = check_fast(got, ref, sample, bank)
    print(name, rep)
    assert rep["cells"] == len(rows) * bank.count
    exact, executed = _device_transform(db, x, n, 2, "exact")
    assert executed == expected_dot_products(bank, n)
    assert exact[torch.from_numpy(rows).cuda()].cpu().numpy().tobytes() == ref.tobytes()
    # every row: PPV integral in l_out, MAX finite (size-independent)
    l_out = torch.from_numpy(bank.output_lengths()).cuda().to(torch.float64)
    for r0 in range(0, n, 8192):
        blk = exact[r0:r0 + 8192]
        counts = blk[:, 0::2].to(torch.float64) * l_out
        assert torch.all((counts - counts.round()).abs() < 1e-3)
        assert torch.isfinite(blk[:, 1::2]).all()


def test_benched_fast_mpv_variant(cuda_ready):
    """bench.py's mpv_fast variant: fast MPV on a 20,000-series config-2
    slice (half-warp MPV chunks), sampled rows vs the oracle with MPV."""
    import torch

    from oracle.oracle import oracle_transform

    bank = generate_bank(1024, 1, 10_000, GenOptions(seed=0))
    n = 20_000
    values = synth_random(n, 1, 1024, seed=1).values
    db = device_bank(bank, 0)
    x = torch.from_numpy(values).cuda()
    rows = np.arange(0, n, 100)
    out, executed = _device_transform(db, x, n, 3, "fast")
    assert executed == expected_dot_products(bank, n)
    ref = oracle_transform(values[rows], bank, include_mpv=True)
    rep = check_fast(out[torch.from_numpy(rows).cuda()].cpu().numpy(), ref, values[rows], bank, fpk=3)
    print(rep)
    exact, _ = _device_transform(db, x, n, 3, "exact")
    assert exact[torch.from_numpy(rows).cuda()].cpu().numpy().tobytes() == ref.tobytes()


@pytest.mark.parametrize("mode", ["fast", "exact"])
def test_pinned_host_pipeline_matches_device_path(mode, cuda_ready):
    """bench.py's e2e call: pinned host x and out, >= 6 row batches through
    the worker pipeline (H2D / kernels / D2H on three streams), a row offset
    and a wider output stride (2-D D2H), fpk 2 and 3, float32 and float64."""
    import torch

    bank = generate_bank(1024, 1, 10_000, GenOptions(seed=0))
    n = 20_000  # >= 4,096 rows -> 6 batches of 3,334
    db = device_bank(bank, 0)
    values = synth_random(n, 1, 1024, seed=1).values
    x_pin = torch.from_numpy(values).pin_memory()
    x_dev = x_pin.cuda()
    for fpk, precision in ((2, "single"), (3, "single"), (2, "double")):
        if precision == "double":
            xp = x_pin.to(torch.float64).pin_memory()
            xd = xp.cuda()
            dt = torch.float64
        else:
            xp, xd, dt = x_pin, x_dev, torch.float32
        ref, _ = _device_transform(db, xd, n, fpk, mode, precision)
        ref = ref.cpu()
        width = bank.count * fpk
        out = torch.full((n + 3, width + 5), float("nan"), dtype=dt).pin_memory()
        executed = db.transform_into(xp.data_ptr(), n, out.data_ptr(), width + 5, row0=3, mode=mode, fpk=fpk,
                                     precision=precision)
        assert executed == expected_dot_products(bank, n)
        assert torch.isnan(out[:3]).all() and torch.isnan(out[:, width:]).all()
        _same(out[3:, :width].contiguous().numpy(), ref.numpy(), fpk, mode, precision)
        # the contiguous case bench.py times
        out2 = torch.empty((n, width), dtype=dt).pin_memory()
        db.transform_into(xp.data_ptr(), n, out2.data_ptr(), width, mode=mode, fpk=fpk, precision=precision)
        _same(out2.numpy(), ref.numpy(), fpk, mode, precision)
        # a geometric batch schedule (small tail batches: 700, 1400, 2800, ...)
        os.environ["RK_E2E_TAIL"] = "700"
        try:
            out2.zero_()
            db.transform_into(xp.data_ptr(), n, out2.data_ptr(), width, mode=mode, fpk=fpk, precision=precision)
        finally:
            del os.environ["RK_E2E_TAIL"]
        _same(out2.numpy(), ref.numpy(), fpk, mode, precision)


def _same(got, ref, fpk, mode, precision):
    """Bytes equal, except fast-mode MPV: its positive sum is reduced in the
    lane order of the chunk layout, which depends on how many series a call
    stages per item (a 3,334-row pipeline batch runs the full-warp twin, a
    20,000-row call the half-warp layout) — PPV and MAX stay bytes-equal,
    MPV agrees to float32 summation rounding."""
    if fpk == 3 and mode == "fast" and precision == "single":
        np.testing.assert_array_equal(got[:, 0::3], ref[:, 0::3])
        np.testing.assert_array_equal(got[:, 1::3], ref[:, 1::3])
        np.testing.assert_allclose(got[:, 2::3], ref[:, 2::3], rtol=1e-5, atol=0)  # MPV_RTOL
    else:
        assert got.tobytes() == ref.tobytes(), (fpk, precision)


@pytest.mark.parametrize("mode", ["fast", "exact"])
def test_public_pageable_transform_matches_device_path(mode, cuda_ready):
    """The public numpy transform() (pageable buffers: the pinned-ring
    pipeline) at 30,000 config-2 rows equals the device-pointer path."""
    import torch

    from paper_2601_17091_b200 import transform

    bank = generate_bank(1024, 1, 10_000, GenOptions(seed=0))
    n = 30_000
    values = synth_random(n, 1, 1024, seed=1).values
    fm = transform(values, bank, mode=mode)
    ref, _ = _device_transform(device_bank(bank, 0), torch.from_numpy(values).cuda(), n, 2, mode)
    assert fm.values.tobytes() == ref.cpu().numpy().tobytes()


@pytest.mark.parametrize("mode", ["fast", "exact"])
def test_run_batch_mode_dropin(mode, cuda_ready):
    """rk_run_batch_f32_mode: the reference's operator argument list plus a
    mode — fast mode reaches the FFMA2 kernels through the drop-in."""
    import ctypes

    from oracle.oracle import oracle_transform

    lib = cuda_ready
    bank = generate_bank(1024, 1, 10_000, GenOptions(seed=0))
    n = 9_000
    x = np.ascontiguousarray(synth_random(n, 1, 1024, seed=1).values)
    out = np.empty((n, bank.count * 2), dtype=np.float32)
    arrs = [np.ascontiguousarray(v) for v in (
        bank.lengths, bank.dilations, bank.paddings, bank.biases.astype(np.float32),
        bank.weights.astype(np.float32), bank.weight_offsets, bank.channel_indices, bank.channel_offsets,
        bank.channel_counts)]
    p = lambda arr: arr.ctypes.data_as(ctypes.c_void_p)  # noqa: E731
    executed = lib.rk_run_batch_f32_mode(p(x), n, 1, 1024, *[p(a) for a in arrs], bank.count, 1024, 2, p(out),
                                         out.shape[1], 0, {"exact": 0, "fast": 1}[mode])
    assert executed == expected_dot_products(bank, n)
    rows = np.arange(0, n, 45)
    ref = oracle_transform(x[rows], bank)
    if mode == "exact":
        assert out[rows].tobytes() == ref.tobytes()
    else:
        check_fast(out[rows], ref, x[rows], bank)
    assert lib.rk_run_batch_f32_mode(p(x), n, 1, 1024, *[p(a) for a in arrs], bank.count, 1024, 2, p(out),
                                     out.shape[1], 0, 7) < 0


def test_default_stream_ordering(cuda_ready):
    """stream=None means the caller's default stream: an asynchronous H2D of
    x queued there must land before the transform reads it, and default-stream
    work queued after the call sees the features (bench config 1's e2e leg)."""
    import torch

    bank = generate_bank(500, 1, 2000, GenOptions(seed=0))
    values = synth_random(3601, 1, 500, seed=1).values
    db = device_bank(bank, 0)
    ref, _ = _device_transform(db, torch.from_numpy(values).cuda(), len(values), 2, "exact")
    x_host = torch.from_numpy(values).pin_memory()
    for _ in range(3):
        xd = x_host.to("cuda", non_blocking=True)  # queued on the default stream
        out = torch.full((len(values), bank.count * 2), float("nan"), device="cuda")
        db.transform_into(xd.data_ptr(), len(values), out.data_ptr(), out.shape[1], mode="exact")
        assert torch.equal(out, ref)  # default-stream comparison after the call


def test_lane_map_orders_agree(monkeypatch, cuda_ready):
    """The run-major lane map only reorders which lane walks which
    run: PPV / MAX bytes equal the residue-major layout's (RK_NO_AMAP=1) in
    both modes, and exact mode equals the oracle (3 channels, L = 2048: the
    config-5 shape, whose d = 3, 5, 7, ... chunks take the run-major map)."""
    import torch

    from oracle.oracle import oracle_transform
    from paper_2601_17091_b200.engine import DeviceBank

    bank = generate_bank(2048, 3, 1500, GenOptions(seed=11))
    n = 600
    values = synth_random(n, 3, 2048, seed=12).values
    x = torch.from_numpy(values).cuda()
    db_run = DeviceBank(bank, 0)
    monkeypatch.setenv("RK_NO_AMAP", "1")
    db_res = DeviceBank(bank, 0)
    assert db_run.info["n_runmajor_chunks"] > 0 and db_res.info["n_runmajor_chunks"] == 0
    for mode in ("fast", "exact"):
        a, ea = _device_transform(db_run, x, n, 2, mode)
        b, eb = _device_transform(db_res, x, n, 2, mode)
        assert ea == eb == expected_dot_products(bank, n)
        assert a.cpu().numpy().tobytes() == b.cpu().numpy().tobytes(), mode
    rows = np.arange(0, n, 25)
    assert a.cpu().numpy()[rows].tobytes() == oracle_transform(values[rows], bank).tobytes()
    db_run.close()
    db_res.close()
