import os
import sys

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TESTS = os.path.dirname(os.path.abspath(__file__))
for p in (REPO, TESTS):
    if p not in sys.path:
        sys.path.insert(0, p)

GOLDEN = os.path.join(TESTS, "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs on the GPU box)")


@pytest.fixture(scope="session")
def golden_transforms():
    with np.load(os.path.join(GOLDEN, "transforms.npz")) as z:
        return {k: z[k] for k in z.files}


@pytest.fixture(scope="session")
def golden_banks():
    import json

    with open(os.path.join(GOLDEN, "banks.json")) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def cuda_ready():
    """Skip-free guard for gpu tests: the library must be built and a GPU
    visible — a missing extension is a failure, not a skip."""
    from paper_2601_17091_b200 import _lib

    lib = _lib.load()
    assert _lib.device_count() >= 1, "no CUDA device visible to the gpu tests"
    return lib
