"""Ridge head vs the reference ridge (golden fixtures from
gridrocket.fit / fit_regression / select_alpha, ridge.py:100-242): float64
agreement to rounding, identical labels and alpha choice.  CPU tests run the
torch head on the CPU; the gpu-marked one on cuda:0."""

import os

import numpy as np
import pytest

from paper_2601_17091_b200 import ridge

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "ridge.npz")


@pytest.fixture(scope="module")
def gold():
    with np.load(GOLD) as z:
        return {k: z[k] for k in z.files}


def _check(g, name, device):
    feats = g[f"{name}/features"]
    labels = [str(v) for v in g["labels"]]
    m = ridge.fit(feats, labels, alpha=1.0, device=device)
    np.testing.assert_allclose(m.weights, g[f"{name}/weights"], rtol=1e-8, atol=1e-11)
    np.testing.assert_allclose(m.intercepts, g[f"{name}/intercepts"], rtol=0, atol=0)
    np.testing.assert_allclose(m.feature_means, g[f"{name}/means"], rtol=1e-12, atol=1e-14)
    np.testing.assert_allclose(m.feature_scales, g[f"{name}/scales"], rtol=1e-12, atol=1e-14)
    assert [int(v) for v in ridge.predict(m, feats, device=device)] == g[f"{name}/predict"].tolist()
    best, scores = ridge.select_alpha(feats, labels, [0.01, 0.1, 1.0, 10.0], seed=4, device=device)
    assert best == g[f"{name}/select_best"][0]
    assert [scores[a] for a in (0.01, 0.1, 1.0, 10.0)] == g[f"{name}/select_scores"].tolist()
    r = ridge.fit_regression(feats, np.arange(feats.shape[0], dtype=np.float64), alpha=0.5, device=device)
    np.testing.assert_allclose(r.weights, g[f"{name}/reg_weights"], rtol=1e-8, atol=1e-10)
    np.testing.assert_allclose(r.intercepts, g[f"{name}/reg_intercepts"])


@pytest.mark.parametrize("name", ["dual", "primal"])
def test_ridge_matches_reference_cpu(gold, name):
    _check(gold, name, "cpu")


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["dual", "primal"])
def test_ridge_matches_reference_gpu(gold, name, cuda_ready):
    _check(gold, name, "cuda")


def test_hand_derived_identity_case():
    """(I + I)^-1 y = [0.5, 0] (reference test_ridge.py:16-20)."""
    w = ridge.solve_penalized(np.eye(2), np.array([1.0, 0.0]), 1.0)
    np.testing.assert_allclose(w.numpy(), [0.5, 0.0], atol=1e-12)


def test_argument_checks():
    with pytest.raises(ValueError):
        ridge.solve_penalized(np.eye(2), np.ones(2), 0.0)
    with pytest.raises(ValueError):
        ridge.fit(np.ones((3, 2)), ["a", "a", "a"], device="cpu")
    with pytest.raises(ValueError):
        ridge.fit(np.array([[np.nan, 1.0], [1.0, 2.0]]), ["a", "b"], device="cpu")
    m = ridge.fit(np.random.default_rng(0).normal(size=(6, 3)), list("ababab"), device="cpu")
    with pytest.raises(ValueError):
        ridge.predict(m, np.ones((2, 4)), device="cpu")
    assert ridge.accuracy(["a", "b"], ["a", "a"]) == 0.5


@pytest.mark.gpu
def test_transform_to_ridge_on_device(cuda_ready):
    """BASELINE config 1 pipeline on the GPU: the transform's features stay in
    HBM and feed the ridge head (SPEC acceptance criterion 6 shape)."""
    import torch

    from paper_2601_17091_b200 import GenOptions, device_bank, generate_bank, synth_two_class

    ds = synth_two_class(200, 128, seed=7)
    bank = generate_bank(128, 1, 10000, GenOptions(seed=0))
    db = device_bank(bank, 0)
    x = torch.from_numpy(ds.values).cuda()
    feats = torch.empty((x.shape[0], 2 * bank.count), device="cuda")
    db.transform_into(x.data_ptr(), x.shape[0], feats.data_ptr(), feats.shape[1], mode="fast",
                      stream=torch.cuda.current_stream().cuda_stream)
    labels = ds.labels
    best, _ = ridge.select_alpha(feats, labels, [0.01, 0.1, 1.0, 10.0], seed=0)
    rng = np.random.Generator(np.random.Philox(key=np.uint64(1)))
    order = rng.permutation(len(labels))
    tr, te = order[:300], order[300:]
    m = ridge.fit(feats[torch.as_tensor(tr, device="cuda")], [labels[i] for i in tr], alpha=best)
    pred = ridge.predict(m, feats[torch.as_tensor(te, device="cuda")])
    assert ridge.accuracy(pred, [labels[i] for i in te]) >= 0.95


FORMATS = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "formats")


@pytest.mark.parametrize("name", ["ridge_cls", "ridge_reg"])
def test_model_file_roundtrip_matches_reference(name, tmp_path):
    """RKRM v1 files the reference's RidgeModel.save wrote
    (tests/golden/make_golden.py:make_ridge_models) load here, re-save byte
    for byte, and a model fitted here on the same features saves a file the
    reference layout reads back to the same fit (float64 rounding)."""
    from paper_2601_17091_b200 import FeatureMatrix, KernelBank
    from paper_2601_17091_b200.binio import FormatError
    from paper_2601_17091_b200.data import load_cache

    path = os.path.join(FORMATS, name + ".rkrm")
    m = ridge.RidgeModel.load(path)
    m.save(tmp_path / "m.rkrm")
    assert (tmp_path / "m.rkrm").read_bytes() == open(path, "rb").read()
    ds = load_cache(os.path.join(FORMATS, "two_class.rkds"))
    feats = FeatureMatrix.load(os.path.join(FORMATS, "two_class_single.rkfm")).values
    assert KernelBank.load(os.path.join(FORMATS, "bank_40x6.rkbk")).count * 2 == feats.shape[1]
    if name == "ridge_cls":
        assert m.class_names == sorted(set(ds.labels))
        ours = ridge.fit(feats, ds.labels, alpha=0.5, device="cpu")
    else:
        assert m.class_names is None
        ours = ridge.fit_regression(feats, np.arange(ds.values.shape[0], dtype=np.float64), alpha=2.0, device="cpu")
    ours.save(tmp_path / "o.rkrm")
    back = ridge.RidgeModel.load(tmp_path / "o.rkrm")
    assert back.alpha == m.alpha and back.class_names == m.class_names
    np.testing.assert_allclose(back.weights, m.weights, rtol=1e-8, atol=1e-11)
    np.testing.assert_allclose(back.intercepts, m.intercepts, rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(back.feature_means, m.feature_means, rtol=1e-12, atol=1e-14)
    np.testing.assert_allclose(back.feature_scales, m.feature_scales, rtol=1e-12, atol=1e-14)
    raw = open(path, "rb").read()
    (tmp_path / "t.rkrm").write_bytes(raw[:-3])
    with pytest.raises(FormatError):
        ridge.RidgeModel.load(tmp_path / "t.rkrm")


@pytest.mark.parametrize("name", ["dual", "primal"])
def test_ridge_oracle_matches_reference(gold, name):
    """The CPU restatement bench.py's config-1 baseline times (oracle/
    ridge_oracle.py) against the reference's own fits."""
    from oracle import ridge_oracle

    feats = gold[f"{name}/features"]
    labels = [str(v) for v in gold["labels"]]
    m = ridge_oracle.fit(feats, labels, alpha=1.0)
    np.testing.assert_allclose(m[0], gold[f"{name}/weights"], rtol=1e-8, atol=1e-11)
    np.testing.assert_allclose(m[1], gold[f"{name}/intercepts"], rtol=0, atol=0)
    assert [int(v) for v in ridge_oracle.predict(m, feats)] == gold[f"{name}/predict"].tolist()
