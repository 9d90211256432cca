"""SPEC.md acceptance criteria exercised on the GPU path (the reference
suite covers them for its CPU engine only, SURVEY.md §4 "Gaps"):
1/2. oracle equivalence and schedule invariance over 100 random
     configurations; 5. PPV single/double divergence only near zero;
6. end-to-end classification accuracy with a ridge head; plus the wide
path's multi-series items."""

import numpy as np
import pytest

import golden_cases as gc
from parity import check_fast
from paper_2601_17091_b200 import (
    GenOptions,
    GridLimits,
    generate_bank,
    synth_random,
    synth_two_class,
    transform,
    transform_sharded,
)

pytestmark = pytest.mark.gpu


def _config(seed):
    rng = np.random.Generator(np.random.Philox(key=np.uint64(seed)))
    n = int(rng.integers(1, 51))
    c = int(rng.integers(1, 5))
    l = int(rng.integers(32, 257))
    k = int(rng.integers(1, 101))
    return rng.standard_normal((n, c, l)), generate_bank(l, c, k, GenOptions(seed=seed + 1))


def test_criterion1_100_random_configs_exact_and_double(cuda_ready):
    from oracle.oracle import oracle_transform

    for seed in range(1000, 1100):
        values, bank = _config(seed)
        single = transform(values, bank).values
        assert single.tobytes() == oracle_transform(values, bank).tobytes(), seed
        double = transform(values, bank, precision="double").values
        assert double.tobytes() == oracle_transform(values, bank, precision="double").tobytes(), seed


def test_criterion2_schedule_invariance(cuda_ready):
    for seed in range(2000, 2020):
        values, bank = _config(seed)
        ref = transform(values, bank).values.tobytes()
        for workers in (1, 2, 16, 1024):
            for max_y in (3, 65535):
                lim = GridLimits(workers_per_cell=workers, max_y=max_y)
                assert transform(values, bank, limits=lim).values.tobytes() == ref
        assert transform_sharded(values, bank, 4).values.tobytes() == ref


def test_criterion5_ppv_divergence_only_near_zero(cuda_ready):
    from oracle.oracle import convolve_f64

    for seed in range(3000, 3050):
        values, bank = _config(seed)
        single = transform(values, bank).values.astype(np.float64)
        double = transform(values, bank, precision="double").values
        m32, m64 = single[:, 1::2], double[:, 1::2]
        assert np.allclose(m32, m64, rtol=1e-4, atol=1e-7)
        for i, k in np.argwhere(single[:, 0::2] != np.float32(double[:, 0::2])):
            v = convolve_f64(values[i], bank, int(k))
            assert np.any(np.abs(v) < 1e-4), (seed, i, k)


def _ridge_fit_predict(xtr, ytr, xte, alpha):
    """Standardised closed-form ridge (dual form, fp64) — test-local head."""
    mu, sd = xtr.mean(0), xtr.std(0)
    sd[sd == 0] = 1.0
    a, b = (xtr - mu) / sd, (xte - mu) / sd
    t = np.where(ytr == 1, 1.0, -1.0)
    coef = a.T @ np.linalg.solve(a @ a.T + alpha * np.eye(a.shape[0]), t - t.mean())
    return (b @ coef + t.mean() > 0).astype(int)


def test_criterion6_end_to_end_classification(cuda_ready):
    ds = synth_two_class(200, 128, seed=7)
    y = np.array([int(v) for v in ds.labels])
    bank = generate_bank(128, 1, 10000, GenOptions(seed=0))
    feats = transform(ds.values, bank, mode="fast").values.astype(np.float64)
    rng = np.random.Generator(np.random.Philox(key=np.uint64(11)))
    order = rng.permutation(len(y))
    tr, va, te = order[:200], order[200:300], order[300:]
    best = max((np.mean(_ridge_fit_predict(feats[tr], y[tr], feats[va], a) == y[va]), a)
               for a in (0.01, 0.1, 1.0, 10.0))
    trva = np.concatenate([tr, va])
    acc = np.mean(_ridge_fit_predict(feats[trva], y[trva], feats[te], best[1]) == y[te])
    assert acc >= 0.95


def test_wide_path_multi_series_items(cuda_ready):
    """n large enough for several series per CTA item (and an odd tail)."""
    from oracle.oracle import oracle_transform

    bank = generate_bank(256, 1, 300, GenOptions(seed=5))
    values = synth_random(8001, 1, 256, seed=3).values
    exact = transform(values, bank).values
    assert exact.tobytes() == oracle_transform(values, bank).tobytes()
    fast = transform(values, bank, mode="fast").values
    check_fast(fast, exact, values, bank)


def test_golden_banks_through_both_modes_agree(golden_transforms, cuda_ready):
    """fast vs exact on the FordA-shape golden slice (tolerance)."""
    case = gc.CASES["forda"]
    values = gc.case_values(case)
    bank = gc.make_bank(gc.BANKS[case["bank"]])
    check_fast(transform(values, bank, mode="fast").values, golden_transforms["forda/single"], values, bank)
