"""CPU tests of the fast-mode tolerance checker (tests/parity.py): it must
accept another correct float evaluation of the same transform, including
cancelling cells that only the float64 certification explains, and reject
real errors."""

import numpy as np
import pytest

from parity import check_fast
from paper_2601_17091_b200 import GenOptions, generate_bank


def _setup(scale, seed=5, n=12, L=300, C=1, K=400):
    bank = generate_bank(L, C, K, GenOptions(seed=seed))
    rng = np.random.default_rng(seed)
    values = (rng.standard_normal((n, C, L)) * scale).astype(np.float32)
    return bank, values


def _other_evaluation(values, bank, fpk=2):
    """A second, differently rounded evaluation: the float64 oracle on the
    float32-cast bank, rounded to float32 at the end."""
    from oracle.oracle import oracle_transform

    b32 = bank
    x64 = values.astype(np.float64)
    orig_w, orig_b = b32.weights, b32.biases
    try:
        b32.weights = orig_w.astype(np.float32).astype(np.float64)
        b32.biases = orig_b.astype(np.float32).astype(np.float64)
        out = oracle_transform(x64, b32, include_mpv=fpk == 3, precision="double")
    finally:
        b32.weights, b32.biases = orig_w, orig_b
    return out.astype(np.float32)


@pytest.mark.parametrize("scale", [1.0, 50.0, 1e-3])
def test_checker_accepts_another_correct_evaluation(scale):
    from oracle.oracle import oracle_transform

    bank, values = _setup(scale)
    ref = oracle_transform(values, bank)
    assert check_fast(ref, ref, values, bank)["max_certified_cells"] == 0
    other = _other_evaluation(values, bank)
    rep = check_fast(other, ref, values, bank)
    assert rep["max_rel_err_uncertified"] <= 1e-5
    ref3 = oracle_transform(values, bank, include_mpv=True)
    check_fast(_other_evaluation(values, bank, fpk=3), ref3, values, bank, fpk=3)


def test_checker_rejects_wrong_max():
    from oracle.oracle import oracle_transform

    bank, values = _setup(1.0)
    ref = oracle_transform(values, bank)
    bad = ref.copy()
    k = int(np.argmax(np.abs(ref[3, 1::2])))
    bad[3, 2 * k + 1] *= 1.0 + 1e-4
    with pytest.raises(AssertionError, match="MAX"):
        check_fast(bad, ref, values, bank)


def test_checker_rejects_wrong_ppv():
    from oracle.oracle import cell_cert, oracle_transform

    bank, values = _setup(1.0)
    ref = oracle_transform(values, bank)
    c = cell_cert(values, bank, np.full(bank.count, 2), np.arange(bank.count))
    k = int(np.flatnonzero(c["unsure"] == 0)[0])
    l_out = bank.output_lengths()[k]
    cnt = int(round(float(ref[2, 2 * k]) * l_out))
    bad = ref.copy()
    bad[2, 2 * k] = np.float32((cnt + 1) / l_out) if cnt < l_out else np.float32((cnt - 1) / l_out)
    with pytest.raises(AssertionError, match="PPV"):
        check_fast(bad, ref, values, bank)


def test_checker_rejects_wrong_mpv():
    from oracle.oracle import oracle_transform

    bank, values = _setup(1.0)
    ref = oracle_transform(values, bank, include_mpv=True)
    bad = ref.copy()
    k = int(np.argmax(ref[1, 2::3]))
    bad[1, 3 * k + 2] *= 1.0 + 1e-3
    with pytest.raises(AssertionError, match="MPV"):
        check_fast(bad, ref, values, bank, fpk=3)


def test_cell_cert_matches_float64_oracle():
    from oracle.oracle import cell_cert, oracle_transform

    bank, values = _setup(1.0, C=3, K=200, n=4)
    c = cell_cert(values, bank, np.repeat(np.arange(4), bank.count), np.tile(np.arange(bank.count), 4))
    ref = _other_evaluation(values, bank).reshape(4, bank.count, 2)
    f32max = ref[:, :, 1].ravel().astype(np.float64)
    assert np.all(np.abs(f32max - c["max64"]) <= np.abs(c["max64"]) * 2 ** -23 + 1e-30)
    l_out = bank.output_lengths()
    counts = np.rint(ref[:, :, 0].astype(np.float64) * l_out).ravel()
    assert np.all(np.abs(counts - c["pos"]) <= c["unsure"])
    assert np.all(c["near"] <= c["unsure"]) and np.all(c["maxerr"] > 0)
