"""Bank generation parity: this package's generate_bank vs reference banks
(fingerprints made by tests/golden/make_golden.py from gridrocket.generate_bank,
reference kernels.py:243-308)."""

import numpy as np
import pytest

import golden_cases as gc
from paper_2601_17091_b200 import (
    GenOptions,
    bank_fingerprint,
    dilation_exponent_bound,
    generate_bank,
    total_positions,
    useful_flops_per_series,
)


@pytest.mark.parametrize("name", sorted(gc.BANKS))
def test_bank_matches_reference(name, golden_banks):
    g = golden_banks["banks"][name]
    bank = gc.make_bank(gc.BANKS[name])
    assert bank_fingerprint(bank) == g["fingerprint"]
    assert bank.lengths[:8].tolist() == g["lengths_head"]
    assert bank.dilations[:8].tolist() == g["dilations_head"]
    assert bank.paddings[:8].tolist() == g["paddings_head"]
    assert bank.biases[:4].tolist() == g["biases_head"]
    assert total_positions(bank) == g["total_positions"]


def test_survey_fingerprint_l1024():
    """SURVEY.md §8c pins sha256(lengths|weights|biases|dilations|paddings)[:16]."""
    import hashlib

    b = generate_bank(1024, 1, 10000, GenOptions(seed=0))
    h = hashlib.sha256()
    for a in (b.lengths, b.weights, b.biases, b.dilations, b.paddings):
        h.update(a.tobytes())
    assert h.hexdigest()[:16] == "b5d8710722623ddf"


@pytest.mark.parametrize(
    "l,c,k,flops",
    [(500, 1, 10000, 81_023_952), (1024, 1, 10000, 169_581_912), (2048, 3, 1000, 47_078_948)],
)
def test_useful_flops_survey_values(l, c, k, flops):
    """Algorithmic FLOPs per series."""
    assert useful_flops_per_series(generate_bank(l, c, k, GenOptions(seed=0))) == flops


def test_formula_values():
    """kernels.py:204-214 known values (reference test_kernels.py:38-40)."""
    assert dilation_exponent_bound(100, 7) == pytest.approx(4.044394119358453)
    assert dilation_exponent_bound(1000, 11) == pytest.approx(6.642412772905056)


def test_same_seed_bit_identical_and_validates():
    a = generate_bank(300, 3, 200, GenOptions(seed=9))
    b = generate_bank(300, 3, 200, GenOptions(seed=9))
    assert bank_fingerprint(a) == bank_fingerprint(b)
    a.validate()
    assert np.all(a.output_lengths() >= 1)
    assert np.all(np.isin(a.channel_counts, [1, 2]))  # floor(2**u), u < log2 3


def test_argument_checks():
    with pytest.raises(ValueError):
        generate_bank(10, 1, 5)
    with pytest.raises(ValueError):
        generate_bank(64, 1, 0)
    with pytest.raises(ValueError):
        generate_bank(64, 0, 5)
