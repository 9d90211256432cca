"""Definitions of the golden parity cases (shared by make_golden.py and the tests).

Inputs are regenerated from seeds with numpy's Philox Generator exactly as
the reference tests do (pkg/tests/conftest.py:7-27, test_engine.py,
test_reference.py); only the reference's outputs are stored
(tests/golden/transforms.npz).
"""

import numpy as np


def _philox(seed):
    return np.random.Generator(np.random.Philox(key=np.uint64(seed)))


def random_config_dims(seed):
    """(n, C, L, K) of the reference's random_config(seed) (conftest.py:7-16)."""
    rng = _philox(seed)
    n = int(rng.integers(1, 51))
    c = int(rng.integers(1, 5))
    l = int(rng.integers(32, 257))
    k = int(rng.integers(1, 101))
    return n, c, l, k


def random_config_values(seed):
    rng = _philox(seed)
    n = int(rng.integers(1, 51))
    c = int(rng.integers(1, 5))
    l = int(rng.integers(32, 257))
    rng.integers(1, 101)
    return rng.standard_normal((n, c, l))


RC_SEEDS = list(range(12)) + [100, 200, 201, 300, 500]

BANKS = {
    "small": ("gen", 64, 1, 20, 11),
    "workers": ("gen", 128, 1, 50, 41),
    "ref13": ("gen", 50, 1, 20, 14),
    "ref15": ("gen", 40, 3, 25, 16),
    "forda": ("gen", 500, 1, 10000, 0),
    "l1024": ("gen", 1024, 1, 10000, 0),
    "mv2048_1k": ("gen", 2048, 3, 1000, 0),
    "mv2048_10k": ("gen", 2048, 3, 10000, 0),
    "l16384": ("gen", 16384, 1, 10000, 0),
    "c8": ("gen", 96, 8, 60, 78),
    "ties": ("gen", 32, 1, 30, 5),
    "zeros": ("custom", "zeros"),
}
for _s in RC_SEEDS:
    _n, _c, _l, _k = random_config_dims(_s)
    BANKS[f"rc{_s}"] = ("gen", _l, _c, _k, _s + 1)

CASES = {
    "small": {"bank": "small", "values": ("philox", 5, (6, 1, 64)),
              "variants": ["single", "double", "single_mpv", "double_mpv"]},
    "workers": {"bank": "workers", "values": ("philox", 40, (20, 1, 128)), "variants": ["single"]},
    "ref13": {"bank": "ref13", "values": ("philox", 13, (10, 1, 50)), "variants": ["single", "double"]},
    "ref15": {"bank": "ref15", "values": ("philox", 15, (6, 3, 40)),
              "variants": ["single", "double_mpv"]},
    "forda": {"bank": "forda", "values": ("synth", 8, 1, 500, 1), "variants": ["single"]},
    "l1024": {"bank": "l1024", "values": ("synth", 8, 1, 1024, 1), "variants": ["single"]},
    "mv2048": {"bank": "mv2048_1k", "values": ("synth", 4, 3, 2048, 1), "variants": ["single"]},
    "l16384": {"bank": "l16384", "values": ("synth", 1, 1, 16384, 1), "variants": ["single"]},
    "c8": {"bank": "c8", "values": ("philox", 77, (5, 8, 96)), "variants": ["single", "double"]},
    "ties": {"bank": "ties", "values": ("zeros", (3, 1, 32)), "variants": ["single", "single_mpv"]},
    "zeros": {"bank": "zeros", "values": ("ones", (3, 1, 32)), "variants": ["single", "double"]},
}
for _s in RC_SEEDS:
    CASES[f"rc{_s}"] = {"bank": f"rc{_s}", "values": ("rc", _s),
                        "variants": ["single", "double"] + (["single_mpv"] if _s < 3 else [])}


def case_values(case):
    kind = case["values"][0]
    if kind == "philox":
        _, seed, shape = case["values"]
        return _philox(seed).standard_normal(shape)
    if kind == "synth":
        _, n, c, l, seed = case["values"]
        return _philox(seed).standard_normal((n, c, l)).astype(np.float32)
    if kind == "rc":
        return random_config_values(case["values"][1])
    if kind == "zeros":
        return np.zeros(case["values"][1])
    if kind == "ones":
        return np.ones(case["values"][1])
    raise ValueError(kind)


def custom_bank_fields(spec):
    """Hand-built banks for edge cases (zero weights, zero / negative-zero
    biases, every length, padded and unpadded)."""
    assert spec == ("custom", "zeros")
    lengths = np.array([7, 9, 11, 7, 9, 11], dtype=np.int32)
    dilations = np.array([1, 2, 3, 4, 1, 2], dtype=np.int32)
    paddings = np.array([3, 0, 15, 0, 4, 10], dtype=np.int32)
    biases = np.array([0.0, 0.5, -0.5, -0.0, 0.25, 1e-30], dtype=np.float64)
    weights = np.zeros(int(lengths.sum()), dtype=np.float64)
    weights[lengths[0] + 2] = 1.0  # kernel 1 sees the series
    return dict(count=6, l_series=32, n_channels=1, lengths=lengths, weights=weights, biases=biases,
                dilations=dilations, paddings=paddings, channel_counts=np.ones(6, dtype=np.int32),
                channel_indices=np.zeros(6, dtype=np.int32), seed=0)


def make_bank(spec):
    """The bank of a spec, built with THIS package's generator."""
    from paper_2601_17091_b200 import GenOptions, KernelBank, generate_bank

    if spec[0] == "gen":
        _, l, c, k, seed = spec
        return generate_bank(l, c, k, GenOptions(seed=seed))
    return KernelBank(**custom_bank_fields(spec))
