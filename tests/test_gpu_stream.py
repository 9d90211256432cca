"""Streaming file transform (rk_transform_stream, paper_2601_17091_b200.
stream) and the CLI on the GPU: feature files must be byte-identical to the
ones the reference wrote (tests/golden/formats/) and to FeatureMatrix.save
of the in-memory transform, across batch splits, shards, input dtypes,
precisions and MPV."""

import os
import subprocess
import sys

import numpy as np
import pytest

from paper_2601_17091_b200 import engine
from paper_2601_17091_b200.data import Dataset, save_cache, synth_random
from paper_2601_17091_b200.features import FeatureMatrix
from paper_2601_17091_b200.kernels import GenOptions, KernelBank, generate_bank
from paper_2601_17091_b200.stream import transform_file

pytestmark = pytest.mark.gpu

FORMATS = os.path.join(os.path.dirname(__file__), "golden", "formats")
REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def golden(name):
    return os.path.join(FORMATS, name)


def read_bytes(path):
    with open(path, "rb") as f:
        return f.read()


@pytest.mark.parametrize(
    "source,kwargs,expect",
    [
        ("two_class.rkds", {}, "two_class_single.rkfm"),
        ("two_class.rkds", {"include_mpv": True}, "two_class_mpv.rkfm"),
        ("two_class.rkds", {"precision": "double"}, "two_class_double.rkfm"),
        ("random64.rkds", {}, "random64_single.rkfm"),
    ],
)
def test_stream_matches_reference_files(cuda_ready, tmp_path, source, kwargs, expect):
    bank = KernelBank.load(golden("bank_40x6.rkbk"))
    stats = transform_file(golden(source), bank, tmp_path / "f.rkfm", **kwargs)
    assert read_bytes(tmp_path / "f.rkfm") == read_bytes(golden(expect))
    n = FeatureMatrix.load(golden(expect)).n_instances
    assert stats.total_dot_products == engine.expected_dot_products(bank, n)


@pytest.mark.parametrize("batch_rows,devices", [(1, 1), (7, 1), (64, 1), (0, 1), (13, 3)])
@pytest.mark.parametrize("mode", ["exact", "fast"])
def test_stream_equals_in_memory(cuda_ready, tmp_path, batch_rows, devices, mode):
    """Batch boundaries and shard splits cannot change a byte."""
    bank = generate_bank(300, 1, 700, GenOptions(seed=11))
    ds = synth_random(301, 1, 300, seed=12)
    save_cache(ds, tmp_path / "d.rkds")
    transform_file(str(tmp_path / "d.rkds"), bank, tmp_path / "s.rkfm", mode=mode, batch_rows=batch_rows,
                   devices=devices)
    engine.transform(ds, bank, mode=mode).save(tmp_path / "m.rkfm")
    assert read_bytes(tmp_path / "s.rkfm") == read_bytes(tmp_path / "m.rkfm")


def test_stream_multichannel_in_memory(cuda_ready, tmp_path):
    bank = generate_bank(96, 3, 200, GenOptions(seed=4))
    values = synth_random(37, 3, 96, seed=5).values
    transform_file(values, bank, tmp_path / "s.rkfm", batch_rows=10, include_mpv=True)
    engine.transform(values, bank, include_mpv=True).save(tmp_path / "m.rkfm")
    assert read_bytes(tmp_path / "s.rkfm") == read_bytes(tmp_path / "m.rkfm")


def test_stream_nonfinite_fails_and_removes_output(cuda_ready, tmp_path):
    bank = generate_bank(64, 1, 50, GenOptions(seed=1))
    values = synth_random(40, 1, 64, seed=2).values.copy()
    values[33, 0, 5] = np.nan
    save_cache(Dataset(values=values), tmp_path / "bad.rkds")
    with pytest.raises(ValueError, match="non-finite"):
        transform_file(str(tmp_path / "bad.rkds"), bank, tmp_path / "f.rkfm", batch_rows=8)
    assert not os.path.exists(tmp_path / "f.rkfm")


def test_stream_shape_errors(cuda_ready, tmp_path):
    bank = generate_bank(64, 1, 50, GenOptions(seed=1))
    save_cache(synth_random(4, 1, 65, seed=2), tmp_path / "d.rkds")
    with pytest.raises(ValueError, match="series length"):
        transform_file(str(tmp_path / "d.rkds"), bank, tmp_path / "f.rkfm")
    with pytest.raises(engine.CapacityError):
        save_cache(synth_random(4, 1, 64, seed=2), tmp_path / "e.rkds")
        transform_file(str(tmp_path / "e.rkds"), bank, tmp_path / "f.rkfm", limits=engine.GridLimits(max_x=10))


def test_stream_empty_dataset(cuda_ready, tmp_path):
    bank = generate_bank(16, 1, 5, GenOptions(seed=1))
    values = np.zeros((0, 1, 16), dtype=np.float32)
    transform_file(values, bank, tmp_path / "f.rkfm")
    FeatureMatrix(values=np.zeros((0, 10), np.float32), n_kernels=5, features_per_kernel=2,
                  precision="single").save(tmp_path / "m.rkfm")
    assert read_bytes(tmp_path / "f.rkfm") == read_bytes(tmp_path / "m.rkfm")


def _cli(*args):
    return subprocess.run([sys.executable, "-m", "paper_2601_17091_b200", *args], cwd=REPO, capture_output=True,
                          text=True, timeout=600)


def test_cli_transform_matches_reference_file(cuda_ready, tmp_path):
    r = _cli("transform", "--data", golden("two_class.rkds"), "--bank", golden("bank_40x6.rkbk"),
             "--out", str(tmp_path / "f.rkfm"), "--csv", str(tmp_path / "f.csv"))
    assert r.returncode == 0, r.stderr
    assert "transformed 6 instances x 12 features (single)" in r.stdout
    assert read_bytes(tmp_path / "f.rkfm") == read_bytes(golden("two_class_single.rkfm"))
    assert read_bytes(tmp_path / "f.csv") == read_bytes(golden("two_class_single.csv"))
    # generated bank (--kernels/--seed) == the saved reference bank
    r = _cli("transform", "--data", golden("two_class.rkds"), "--kernels", "6", "--seed", "5", "--precision",
             "double", "--devices", "2", "--out", str(tmp_path / "g.rkfm"))
    assert r.returncode == 0, r.stderr
    assert read_bytes(tmp_path / "g.rkfm") == read_bytes(golden("two_class_double.rkfm"))


def test_cli_exit_codes(cuda_ready, tmp_path):
    r = _cli("transform", "--data", golden("two_class.rkds"), "--out", str(tmp_path / "f.rkfm"))
    assert r.returncode == 2 and "either --bank or --kernels" in r.stderr
    r = _cli("transform", "--data", golden("two_class.rkds"), "--kernels", "6", "--max-x", "3",
             "--out", str(tmp_path / "f.rkfm"))
    assert r.returncode == 3
    r = _cli("transform", "--data", golden("two_class.rkds"), "--kernels", "6", "--memory-budget", "16",
             "--out", str(tmp_path / "f.rkfm"))
    assert r.returncode == 3 and "capacity error" in r.stderr
