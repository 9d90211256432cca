"""Native bank generation (rk_generate_bank, csrc/bank_gen.cpp, SURVEY.md
§8 f4) against the numpy draw path and the reference's golden bank
fingerprints: every field bit-identical.  Host-only (no GPU)."""

import json
import os

import numpy as np
import pytest

from paper_2601_17091_b200.kernels import GenOptions, bank_fingerprint, generate_bank

FIELDS = ("lengths", "weights", "biases", "dilations", "paddings", "channel_counts", "channel_indices")
GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "banks.json")


def same(a, b):
    return all(getattr(a, f).dtype == getattr(b, f).dtype and getattr(a, f).tobytes() == getattr(b, f).tobytes()
               for f in FIELDS)


@pytest.mark.parametrize(
    "l_series,n_channels,count,seed,center",
    [
        (1024, 1, 10000, 0, True),     # BASELINE config 2 bank
        (500, 1, 3000, 3, True),
        (16384, 1, 1500, 2, True),     # config 4 length
        (2048, 3, 3000, 1, True),      # config 5 shape
        (64, 7, 2000, 9, False),       # uncentred, odd channel count
        (11, 1, 400, 5, True),         # shortest series: every dilation is 1
        (300, 64, 300, 4, True),       # Floyd's algorithm over many channels
        (100, 12000, 12, 7, True),     # > 10000 channels: tail-shuffle choice
        (40, 2, 1000, 123456789012, True),
        (77, 5, 700, 2**64 - 1, True),  # largest key
    ],
)
def test_native_equals_numpy(l_series, n_channels, count, seed, center):
    opts = GenOptions(seed=seed, center_weights=center)
    a = generate_bank(l_series, n_channels, count, opts, native=False)
    b = generate_bank(l_series, n_channels, count, opts, native=True)
    assert same(a, b)


def test_native_matches_reference_fingerprints():
    with open(GOLDEN) as f:
        banks = json.load(f)["banks"]
    checked = 0
    for name, entry in banks.items():
        spec = entry["spec"]
        if spec[0] != "gen":
            continue
        _, l_series, n_channels, count, seed = spec
        bank = generate_bank(l_series, n_channels, count, GenOptions(seed=seed), native=True)
        assert bank_fingerprint(bank) == entry["fingerprint"], name
        checked += 1
    assert checked >= 3


def test_native_default_and_errors():
    from paper_2601_17091_b200 import _lib

    bank = generate_bank(1024, 1, 5, GenOptions(seed=0))
    assert bank.lengths.tolist() == [7, 7, 11, 7, 9] and bank.dilations.tolist() == [2, 9, 3, 10, 72]
    with pytest.raises(OverflowError):
        generate_bank(64, 1, 3, GenOptions(seed=-1), native=True)
    lib = _lib.load()
    assert lib.rk_generate_bank(0, 64, 1, 0, 1, None, 0.0, *([None] * 6), 0, None, 0, None, None) == \
        _lib.RK_ERR_INVALID


def test_native_capacity_retry_reports_sizes():
    """A too-small buffer gets RK_ERR_CAPACITY with the exact sizes needed
    (the caller's retry then yields the same bank as numpy)."""
    import ctypes

    from paper_2601_17091_b200 import _lib
    from paper_2601_17091_b200.kernels import CANDIDATE_LENGTHS, dilation_exponent_bound

    lib = _lib.load()
    count, L, C = 50, 64, 40
    bounds = np.array([dilation_exponent_bound(L, lk) for lk in CANDIDATE_LENGTHS], dtype=np.float64)
    outs = [np.empty(count, np.int32), np.empty(count), np.empty(count, np.int32), np.empty(count, np.int32),
            np.empty(count, np.int32)]
    idx = np.empty(1, np.int32)
    w = np.empty(1)
    n_w, n_i = ctypes.c_int64(0), ctypes.c_int64(0)
    p = lambda a: a.ctypes.data_as(ctypes.c_void_p)  # noqa: E731
    rc = lib.rk_generate_bank(count, L, C, ctypes.c_uint64(9), 1, p(bounds), float(np.log2(C)), *[p(a) for a in outs],
                              p(idx), idx.size, p(w), w.size, ctypes.byref(n_w), ctypes.byref(n_i))
    assert rc == _lib.RK_ERR_CAPACITY
    ref = generate_bank(L, C, count, GenOptions(seed=9), native=False)
    assert n_i.value == ref.channel_indices.size and n_w.value == ref.weights.size
    nat = generate_bank(L, C, count, GenOptions(seed=9), native=True)
    assert nat.weights.tobytes() == ref.weights.tobytes()
    assert nat.channel_indices.tobytes() == ref.channel_indices.tobytes()
