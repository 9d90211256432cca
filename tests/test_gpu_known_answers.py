"""Known-answer and invariant tests of the reference (pkg/tests/
test_reference.py:59-184: apply_kernel cases, bias shift, power-of-two
scaling, identical rows, MPV iff PPV) restated for the CUDA transform with
hand-built banks, in both modes."""

import numpy as np
import pytest

from paper_2601_17091_b200 import KernelBank, transform

pytestmark = pytest.mark.gpu


def bank_of(weights, biases, dilations, paddings, l_series):
    weights = [np.asarray(w, dtype=np.float64) for w in weights]
    k = len(weights)
    return KernelBank(
        count=k, l_series=l_series, n_channels=1,
        lengths=[len(w) for w in weights], weights=np.concatenate(weights), biases=biases,
        dilations=dilations, paddings=paddings, channel_counts=[1] * k, channel_indices=[0] * k, seed=0,
    )


@pytest.mark.parametrize("mode", ["exact", "fast"])
def test_apply_kernel_cases(mode, cuda_ready):
    """All-negative outputs, a bias that makes every output positive, and
    all-zero outputs (test_reference.py:59-80)."""
    series = np.arange(16, dtype=np.float32)[None, None, :]
    bank = bank_of([[-1.0] * 7, [1.0] * 7, [0.0] * 7], [0.0, 2.0, 0.0], [1, 1, 1], [0, 0, 0], 16)
    out = transform(series, bank, include_mpv=True, mode=mode).values[0]
    # kernel 0: -(sum of 7 consecutive values) < 0 everywhere; max at t = 0
    assert out[0] == 0.0 and out[1] == -21.0 and out[2] == 0.0
    # kernel 1: sum + 2 > 0 everywhere; max at the last window: 9+...+15 + 2
    assert out[3] == 1.0 and out[4] == 86.0
    # kernel 2: zero weights, zero bias: no positives, max 0, mpv 0
    assert out[6] == 0.0 and out[7] == 0.0 and out[8] == 0.0


@pytest.mark.parametrize("mode", ["exact", "fast"])
def test_bias_shift_and_power_of_two_scaling(mode, cuda_ready):
    """MAX moves by exactly the bias (RN(max acc + b)) and scales exactly
    with power-of-two inputs; PPV is monotone in the bias and invariant
    under scaling (test_reference.py:139-174)."""
    rng = np.random.Generator(np.random.Philox(key=np.uint64(31)))
    series = rng.standard_normal((3, 1, 60)).astype(np.float32)
    w9 = rng.standard_normal(9)
    w7 = rng.standard_normal(7)
    w11 = rng.standard_normal(11)

    def run(x, bias):
        bank = bank_of([w9, w7, w11], [bias] * 3, [3, 2, 1], [0, 6, 5], 60)
        return transform(x, bank, mode=mode).values

    base = run(series, 0.0)
    for shift in (0.5, 1.25, 2.0):
        moved = run(series, shift)
        expect = (base[:, 1::2] + np.float32(shift)).astype(np.float32)
        if mode == "exact":
            assert np.array_equal(moved[:, 1::2], expect)
        else:
            assert np.allclose(moved[:, 1::2], expect, rtol=1e-5, atol=1e-6)
        assert np.all(moved[:, 0::2] >= base[:, 0::2])
    for s in (0.5, 2.0, 4.0):
        scaled = run(series * np.float32(s), 0.0)
        assert np.array_equal(scaled[:, 1::2], base[:, 1::2] * np.float32(s))
        assert np.array_equal(scaled[:, 0::2], base[:, 0::2])


@pytest.mark.parametrize("mode", ["exact", "fast"])
def test_identical_series_identical_rows_and_mpv_iff_ppv(mode, cuda_ready):
    """Identical series give identical rows; MPV > 0 exactly when PPV > 0
    (test_reference.py:82-91, 110-114)."""
    from paper_2601_17091_b200 import GenOptions, generate_bank

    bank = generate_bank(64, 1, 500, GenOptions(seed=2))
    series = np.tile(np.linspace(-1, 1, 64, dtype=np.float32), (4, 1, 1))
    out = transform(series, bank, include_mpv=True, mode=mode).values
    assert all(np.array_equal(out[0], out[i]) for i in range(1, 4))
    rng = np.random.Generator(np.random.Philox(key=np.uint64(21)))
    x = rng.standard_normal((20, 1, 64)).astype(np.float32)
    out = transform(x, bank, include_mpv=True, mode=mode).values
    ppv, mpv = out[:, 0::3], out[:, 2::3]
    assert np.all(mpv >= 0.0)
    assert np.array_equal(mpv > 0.0, ppv > 0.0)
