"""Series longer than one CTA's shared memory (the reference has no such
limit): the wide kernel's GMEM variants read the windows from zero-haloed
rows in global memory.  Exact bytes against the oracle, fast tolerance, and
the float64 / MPV cell paths, for single-channel and EigenWorms-like
(6 channels x 17,984) shapes."""

import numpy as np
import pytest

from parity import check_fast
from paper_2601_17091_b200 import GenOptions, device_bank, generate_bank, synth_random, transform

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("l_series,n_channels,count,n", [(40_000, 1, 300, 3), (17_984, 6, 120, 2),
                                                         (65_536, 1, 60, 2)])
def test_long_series_exact_and_fast(l_series, n_channels, count, n, cuda_ready):
    from oracle.oracle import oracle_transform

    bank = generate_bank(l_series, n_channels, count, GenOptions(seed=7))
    assert device_bank(bank).info["path"] == 2  # wide kernel, series in global memory
    values = synth_random(n, n_channels, l_series, seed=8).values
    ref = oracle_transform(values, bank)
    assert transform(values, bank, mode="exact").values.tobytes() == ref.tobytes()
    check_fast(transform(values, bank, mode="fast").values, ref, values, bank)


@pytest.mark.parametrize("l_series", [30_000, 70_000])
def test_long_series_mpv_and_double(l_series, cuda_ready):
    """Exact MPV and float64 run the cell kernels (unstaged beyond shared
    memory): bytes equal; fast MPV within its tolerance."""
    from oracle.oracle import oracle_transform

    bank = generate_bank(l_series, 1, 40, GenOptions(seed=9))
    values = synth_random(2, 1, l_series, seed=10).values
    mpv_ref = oracle_transform(values, bank, include_mpv=True)
    assert transform(values, bank, include_mpv=True).values.tobytes() == mpv_ref.tobytes()
    check_fast(transform(values, bank, include_mpv=True, mode="fast").values, mpv_ref, values, bank, fpk=3)
    dbl = transform(values, bank, precision="double").values
    assert dbl.tobytes() == oracle_transform(values, bank, precision="double").tobytes()


def test_long_series_many_rows_batches(cuda_ready):
    """More rows than one 1 GB batch of padded rows: the chain runs per
    batch with fresh item counters."""
    from oracle.oracle import oracle_transform

    bank = generate_bank(60_000, 1, 8, GenOptions(seed=11))
    values = synth_random(1200, 1, 60_000, seed=12).values  # ~1.2k rows x 240 KB padded > 1 GB
    out = transform(values, bank, mode="exact").values
    rows = [0, 1, 599, 1000, 1199]
    assert out[rows].tobytes() == oracle_transform(values[rows], bank).tobytes()
