"""Pin the CPU oracle (oracle/rocket_oracle.c) to the reference: its output
must be byte-identical to gridrocket.transform's on every golden case
(single and double precision, with and without MPV)."""

import numpy as np
import pytest

import golden_cases as gc
from oracle.oracle import convolve_f64, oracle_transform

VARIANTS = [(name, v) for name, case in gc.CASES.items() for v in case["variants"]]


@pytest.mark.parametrize("name,variant", VARIANTS)
def test_oracle_matches_reference(name, variant, golden_transforms):
    case = gc.CASES[name]
    values = gc.case_values(case)
    bank = gc.make_bank(gc.BANKS[case["bank"]])
    precision = variant.split("_")[0]
    mpv = variant.endswith("_mpv")
    out, executed = oracle_transform(values, bank, include_mpv=mpv, precision=precision,
                                     return_executed=True)
    expected = golden_transforms[f"{name}/{variant}"]
    assert out.dtype == expected.dtype and out.shape == expected.shape
    assert out.tobytes() == expected.tobytes()
    assert executed == int(golden_transforms[f"{name}/{variant}/executed"][0])


def test_oracle_thread_count_invariant():
    case = gc.CASES["rc3"]
    values = gc.case_values(case)
    bank = gc.make_bank(gc.BANKS[case["bank"]])
    a = oracle_transform(values, bank, nthreads=1)
    b = oracle_transform(values, bank, nthreads=7)
    assert a.tobytes() == b.tobytes()


def test_convolve_f64_matches_double_max(golden_transforms):
    case = gc.CASES["small"]
    values = gc.case_values(case)
    bank = gc.make_bank(gc.BANKS["small"])
    ref = golden_transforms["small/double"]
    for k in range(bank.count):
        v = convolve_f64(values[0], bank, k)
        assert v.max() == ref[0, 2 * k + 1]
        assert np.float64(np.count_nonzero(v > 0)) / v.shape[0] == ref[0, 2 * k]
