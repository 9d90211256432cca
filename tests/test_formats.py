"""File formats against files the reference itself wrote
(tests/golden/formats/, made by tests/golden/make_golden.py:make_formats):
bank (RKBK), dataset cache (RKDS), feature matrix (RKFM) and its CSV export,
and the reference's own data / feature / bank test cases
(/root/reference/pkg/tests/test_data.py, test_features.py,
test_kernels.py:160-195) restated."""

import os

import numpy as np
import pytest

from paper_2601_17091_b200.binio import FormatError
from paper_2601_17091_b200.data import (
    Dataset,
    cache_layout,
    load_cache,
    load_dataset,
    read_cache_labels,
    save_cache,
    synth_random,
    synth_two_class,
)
from paper_2601_17091_b200.features import FEATURE_DATA_OFFSET, FeatureMatrix
from paper_2601_17091_b200.kernels import GenOptions, KernelBank, generate_bank

FORMATS = os.path.join(os.path.dirname(__file__), "golden", "formats")


def golden(name):
    return os.path.join(FORMATS, name)


def read_bytes(path):
    with open(path, "rb") as f:
        return f.read()


# ---- writers reproduce the reference's bytes --------------------------------

def test_bank_file_bytes(tmp_path):
    generate_bank(40, 1, 6, GenOptions(seed=5)).save(tmp_path / "b.rkbk")
    assert read_bytes(tmp_path / "b.rkbk") == read_bytes(golden("bank_40x6.rkbk"))
    generate_bank(32, 3, 4, GenOptions(seed=6, center_weights=False)).save(tmp_path / "c.rkbk")
    assert read_bytes(tmp_path / "c.rkbk") == read_bytes(golden("bank_3ch.rkbk"))


def test_bank_file_load_roundtrip():
    bank = KernelBank.load(golden("bank_3ch.rkbk"))
    ref = generate_bank(32, 3, 4, GenOptions(seed=6, center_weights=False))
    assert bank.center_weights is False and bank.seed == 6
    for field in ("lengths", "weights", "biases", "dilations", "paddings", "channel_counts", "channel_indices"):
        assert getattr(bank, field).tobytes() == getattr(ref, field).tobytes()


def test_cache_bytes(tmp_path):
    save_cache(synth_two_class(3, 40, seed=8), tmp_path / "d.rkds")
    assert read_bytes(tmp_path / "d.rkds") == read_bytes(golden("two_class.rkds"))
    ds64 = Dataset(values=synth_random(4, 1, 40, seed=9).values.astype(np.float64) * 1.5, name="random64")
    save_cache(ds64, tmp_path / "r.rkds")
    assert read_bytes(tmp_path / "r.rkds") == read_bytes(golden("random64.rkds"))


@pytest.mark.parametrize("name", ["two_class_single", "two_class_mpv", "two_class_double", "random64_single"])
def test_feature_file_roundtrip_bytes(tmp_path, name):
    fm = FeatureMatrix.load(golden(name + ".rkfm"))
    fm.save(tmp_path / "f.rkfm")
    assert read_bytes(tmp_path / "f.rkfm") == read_bytes(golden(name + ".rkfm"))
    assert fm.values.dtype == (np.float64 if "double" in name else np.float32)
    assert fm.features_per_kernel == (3 if "mpv" in name else 2)


@pytest.mark.parametrize("name", ["two_class_single", "two_class_double"])
def test_feature_csv_bytes(tmp_path, name):
    FeatureMatrix.load(golden(name + ".rkfm")).to_csv(tmp_path / "f.csv")
    assert read_bytes(tmp_path / "f.csv") == read_bytes(golden(name + ".csv"))


# ---- readers ----------------------------------------------------------------

def test_cache_layout_and_labels():
    layout = cache_layout(golden("two_class.rkds"))
    ds = load_cache(golden("two_class.rkds"))
    assert (layout.n_instances, layout.n_channels, layout.l_series) == ds.values.shape
    assert layout.dtype == np.float32 and layout.has_labels and layout.name == "synth_two_class"
    raw = read_bytes(golden("two_class.rkds"))
    block = np.frombuffer(raw[layout.values_offset : layout.values_offset + layout.values_bytes], "<f4")
    assert block.tobytes() == ds.values.tobytes()
    assert read_cache_labels(golden("two_class.rkds"), layout) == ds.labels
    assert ds.values.tobytes() == synth_two_class(3, 40, seed=8).values.tobytes()
    lay64 = cache_layout(golden("random64.rkds"))
    assert lay64.dtype == np.float64 and not lay64.has_labels
    assert read_cache_labels(golden("random64.rkds"), lay64) is None


def test_load_dataset_dispatch(tmp_path):
    c = load_dataset(golden("two_class.rkds"))
    assert c.name == "synth_two_class" and c.labels == synth_two_class(3, 40, seed=8).labels
    np.save(tmp_path / "d.npy", c.values)
    assert load_dataset(tmp_path / "d.npy").values.tobytes() == c.values.tobytes()
    # text ingestion is out of scope: a clear error, not a parse
    for name in ("two_class.ts", "two_class.csv"):
        with pytest.raises(ValueError, match="not read by this package"):
            load_dataset(golden(name))


def test_truncated_files_raise_format_error(tmp_path):
    for name in ("two_class.rkds", "bank_40x6.rkbk", "two_class_single.rkfm"):
        raw = read_bytes(golden(name))
        (tmp_path / name).write_bytes(raw[: len(raw) - 5])
    with pytest.raises(FormatError):
        load_cache(tmp_path / "two_class.rkds")
    with pytest.raises(FormatError):
        KernelBank.load(tmp_path / "bank_40x6.rkbk")
    with pytest.raises(FormatError):
        FeatureMatrix.load(tmp_path / "two_class_single.rkfm")
    with pytest.raises(FormatError):
        cache_layout_path = tmp_path / "short.rkds"
        cache_layout_path.write_bytes(read_bytes(golden("two_class.rkds"))[:100])
        cache_layout(cache_layout_path)


def test_bad_magic_and_version(tmp_path):
    raw = bytearray(read_bytes(golden("two_class_single.rkfm")))
    (tmp_path / "m.rkfm").write_bytes(b"XXXX" + bytes(raw[4:]))
    with pytest.raises(FormatError):
        FeatureMatrix.load(tmp_path / "m.rkfm")
    raw[4:8] = (2).to_bytes(4, "little")
    (tmp_path / "v.rkfm").write_bytes(bytes(raw))
    with pytest.raises(FormatError):
        FeatureMatrix.load(tmp_path / "v.rkfm")
    assert FEATURE_DATA_OFFSET == 29


# ---- the reference's data tests (test_data.py) ------------------------------

def test_dataset_invariants():
    with pytest.raises(ValueError):
        Dataset(values=np.zeros((2, 1, 4)), labels=["only-one"])
    with pytest.raises(ValueError):
        Dataset(values=np.zeros((2, 4)))
