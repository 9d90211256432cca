"""Host-side logic (no GPU): plans, accumulators, validation, containers —
the reference's own known answers (pkg/tests/test_engine.py:26-115)."""

import numpy as np
import pytest
from hypothesis import given, settings
from hypothesis import strategies as st

from paper_2601_17091_b200 import (
    CapacityError,
    FeatureMatrix,
    GenOptions,
    GridLimits,
    bytes_per_instance,
    expected_dot_products,
    generate_bank,
    plan_batches,
    plan_shards,
    reduce_cell,
    total_positions,
)
from paper_2601_17091_b200.engine import _check_shapes


def test_grid_y_limit_looping():
    plan = plan_batches(70000, 100, GridLimits(memory_budget_bytes=1 << 40))
    assert [c for _, c in plan.batches] == [65535, 4465]
    assert plan.batches[1] == (65535, 4465)


def test_memory_bound_batches():
    plan = plan_batches(100, 10, GridLimits(memory_budget_bytes=79))
    assert [c for _, c in plan.batches] == [7] * 14 + [2]


def test_instance_too_large():
    with pytest.raises(CapacityError):
        plan_batches(5, 1000, GridLimits(memory_budget_bytes=999))


@given(n=st.integers(0, 5000), bpi=st.integers(1, 64), max_y=st.integers(1, 512), units=st.integers(1, 2048))
@settings(max_examples=60, deadline=None)
def test_batches_partition(n, bpi, max_y, units):
    plan = plan_batches(n, bpi, GridLimits(max_y=max_y, memory_budget_bytes=bpi * units))
    cursor = 0
    for start, count in plan.batches:
        assert start == cursor and 1 <= count <= min(max_y, units)
        cursor += count
    assert cursor == n


def test_shards():
    assert [c for _, c in plan_shards(10, 3)] == [4, 3, 3]
    assert [c for _, c in plan_shards(2, 3)] == [1, 1, 0]
    with pytest.raises(ValueError):
        plan_shards(5, 0)


@given(n=st.integers(0, 10000), k=st.integers(1, 64))
@settings(max_examples=60, deadline=None)
def test_shards_balanced(n, k):
    sizes = [c for _, c in plan_shards(n, k)]
    assert sum(sizes) == n and max(sizes) - min(sizes) <= 1


def test_reduce_cell_monoid():
    acc = reduce_cell([(True, 1.0), (False, -1.0), (True, 2.0)])
    assert (acc.ppv_count, acc.running_max) == (2, 2.0)
    empty = reduce_cell([])
    assert (empty.ppv_count, empty.running_max) == (0, float("-inf"))
    left, right = reduce_cell([(True, 0.5), (False, -2.0)]), reduce_cell([(True, 3.5)])
    merged = left.merge(right)
    assert (merged.ppv_count, merged.running_max) == (2, 3.5)


def test_limits_and_formulas():
    with pytest.raises(ValueError):
        GridLimits(max_y=0)
    assert bytes_per_instance(3, 1000) == 12000
    bank = generate_bank(64, 1, 20, GenOptions(seed=11))
    assert expected_dot_products(bank, 6) == 6 * total_positions(bank)


def test_check_shapes_errors():
    bank = generate_bank(64, 1, 20, GenOptions(seed=11))
    with pytest.raises(ValueError):
        _check_shapes(np.zeros((2, 2, 64)), bank, GridLimits())
    with pytest.raises(ValueError):
        _check_shapes(np.zeros((2, 1, 32)), bank, GridLimits())
    bad = np.zeros((2, 1, 64))
    bad[1, 0, 5] = np.nan
    with pytest.raises(ValueError):
        _check_shapes(bad, bank, GridLimits())
    with pytest.raises(CapacityError):
        _check_shapes(np.zeros((2, 1, 64)), bank, GridLimits(max_x=3))


def test_feature_matrix_layout():
    fm = FeatureMatrix(values=np.arange(12, dtype=np.float32).reshape(2, 6), n_kernels=3,
                       features_per_kernel=2, precision="single")
    assert fm.feature("ppv").tolist() == [[0, 2, 4], [6, 8, 10]]
    assert fm.feature("max").tolist() == [[1, 3, 5], [7, 9, 11]]
    assert fm.column_names()[:2] == ["k0_ppv", "k0_max"]
    with pytest.raises(ValueError):
        fm.feature("mpv")
    with pytest.raises(ValueError):
        FeatureMatrix(values=np.zeros((2, 5)), n_kernels=3, features_per_kernel=2, precision="single")


def test_transform_fails_loudly_without_gpu():
    """The product path has no CPU fallback."""
    from paper_2601_17091_b200 import _lib, transform

    if _lib.device_count() > 0:
        pytest.skip("a GPU is visible")
    bank = generate_bank(64, 1, 20, GenOptions(seed=11))
    with pytest.raises((RuntimeError, OSError)):
        transform(np.zeros((2, 1, 64)), bank)


def test_ppv_single_rounding_equals_double_rounding():
    """The kernels compute PPV as RN32(count / l_out) (transform_kernel.cuh,
    finish_chunk); the reference stores f32(RN64(count / l_out))
    (engine.py:187).  Equal for every count <= l_out < 2^24: exhaustive
    for l_out <= 20000, sampled above."""
    import numpy as np

    for n in range(1, 20001):
        c = np.arange(0, n + 1, dtype=np.int64)
        a = (c.astype(np.float64) / n).astype(np.float32)
        b = c.astype(np.float32) / np.float32(n)
        assert np.array_equal(a.view(np.uint32), b.view(np.uint32)), n
    rng = np.random.default_rng(0)
    for _ in range(50):
        n = int(rng.integers(20001, 1 << 24))
        c = np.concatenate([rng.integers(0, n + 1, size=100000), [0, 1, n - 1, n]])
        a = (c.astype(np.float64) / n).astype(np.float32)
        b = c.astype(np.float32) / np.float32(n)
        assert np.array_equal(a.view(np.uint32), b.view(np.uint32)), n
