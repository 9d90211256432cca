"""Generate the golden fixtures from the reference implementation.

Run HERE (the container that mounts /root/reference); the outputs are
committed under tests/golden/ so the GPU box, which has no /root/reference,
can check parity:

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden.py

Fixtures:
  banks.json      fingerprints of reference banks (gridrocket.generate_bank,
                  kernels.py:243-308) for every bank the tests use;
  transforms.npz  reference features (gridrocket.transform, engine.py:324-333,
                  precision single/double, with and without MPV) for seeded
                  inputs; inputs are regenerated from their seeds by
                  tests/golden_cases.py, which defines the cases.
"""

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.join(REPO, "tests"))
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

import gridrocket as gr  # noqa: E402

import golden_cases as gc  # noqa: E402


def fingerprint(bank):
    import hashlib

    h = hashlib.sha256()
    for arr in (bank.lengths, bank.weights, bank.biases, bank.dilations, bank.paddings,
                bank.channel_counts, bank.channel_indices):
        h.update(np.ascontiguousarray(arr).tobytes())
    return h.hexdigest()[:16]


def survey_fingerprint(bank):
    import hashlib

    h = hashlib.sha256()
    for arr in (bank.lengths, bank.weights, bank.biases, bank.dilations, bank.paddings):
        h.update(np.ascontiguousarray(arr).tobytes())
    return h.hexdigest()[:16]


def ref_bank(spec):
    if spec[0] == "gen":
        _, l, c, k, seed = spec
        return gr.generate_bank(l, c, k, gr.GenOptions(seed=seed))
    fields = gc.custom_bank_fields(spec)
    return gr.KernelBank(**fields)


def main():
    banks = {}
    for name, spec in gc.BANKS.items():
        b = ref_bank(spec)
        banks[name] = {
            "spec": list(spec),
            "fingerprint": fingerprint(b),
            "survey_fingerprint": survey_fingerprint(b),
            "count": int(b.count),
            "lengths_head": b.lengths[:8].tolist(),
            "dilations_head": b.dilations[:8].tolist(),
            "paddings_head": b.paddings[:8].tolist(),
            "biases_head": b.biases[:4].tolist(),
            "total_positions": int(gr.engine.total_positions(b)),
        }
        print(name, banks[name]["fingerprint"], flush=True)
    with open(os.path.join(HERE, "banks.json"), "w") as f:
        json.dump({"numpy": np.__version__, "banks": banks}, f, indent=1)

    arrays = {}
    for name, case in gc.CASES.items():
        values = gc.case_values(case)
        bank = ref_bank(gc.BANKS[case["bank"]])
        for variant in case["variants"]:
            mpv = variant.endswith("_mpv")
            precision = variant.split("_")[0]
            fm, stats = gr.transform_with_stats(values, bank, include_mpv=mpv, precision=precision)
            arrays[f"{name}/{variant}"] = fm.values
            arrays[f"{name}/{variant}/executed"] = np.array([stats.total_dot_products], dtype=np.int64)
        print(name, values.shape, flush=True)
    np.savez_compressed(os.path.join(HERE, "transforms.npz"), **arrays)
    make_ridge()
    make_formats()
    make_ridge_models()


def make_ridge():
    """Reference ridge fits (ridge.py:100-242) on reference features of the
    labelled fixture: a dual (features > rows) and a primal case, a
    regression and an alpha selection."""
    out = {}
    ds = gr.synth_two_class(30, 64, seed=3)
    labels = np.array(ds.labels)
    for name, k in (("dual", 200), ("primal", 10)):
        bank = gr.generate_bank(64, 1, k, gr.GenOptions(seed=0))
        feats = gr.transform(ds, bank).values
        m = gr.fit(feats, labels, alpha=1.0)
        out[f"{name}/features"] = feats
        out[f"{name}/weights"] = m.weights
        out[f"{name}/intercepts"] = m.intercepts
        out[f"{name}/means"] = m.feature_means
        out[f"{name}/scales"] = m.feature_scales
        out[f"{name}/predict"] = gr.predict(m, feats).astype(np.int64)
        best, scores = gr.select_alpha(feats, labels, [0.01, 0.1, 1.0, 10.0], seed=4)
        out[f"{name}/select_best"] = np.array([best])
        out[f"{name}/select_scores"] = np.array([scores[a] for a in (0.01, 0.1, 1.0, 10.0)])
        r = gr.fit_regression(feats, np.arange(feats.shape[0], dtype=np.float64), alpha=0.5)
        out[f"{name}/reg_weights"] = r.weights
        out[f"{name}/reg_intercepts"] = r.intercepts
    out["labels"] = labels.astype(np.int64)
    np.savez_compressed(os.path.join(HERE, "ridge.npz"), **out)


def make_formats():
    """Files written by the reference's own writers (_binio.py, kernels.py:
    127-147, data.py:193-276, features.py:59-91) for the format parity
    tests: a bank, dataset caches (f32 with labels, f64 without), and
    feature files of reference transforms of the cached
    dataset (single / single+MPV / double) plus one CSV export."""
    from gridrocket.data import save_cache

    out = os.path.join(HERE, "formats")
    os.makedirs(out, exist_ok=True)
    bank = gr.generate_bank(40, 1, 6, gr.GenOptions(seed=5))
    bank.save(os.path.join(out, "bank_40x6.rkbk"))
    gr.generate_bank(32, 3, 4, gr.GenOptions(seed=6, center_weights=False)).save(
        os.path.join(out, "bank_3ch.rkbk"))
    ds = gr.synth_two_class(3, 40, seed=8)
    save_cache(ds, os.path.join(out, "two_class.rkds"))
    ds64 = gr.Dataset(values=gr.synth_random(4, 1, 40, seed=9).values.astype(np.float64) * 1.5,
                      name="random64")
    save_cache(ds64, os.path.join(out, "random64.rkds"))
    gr.transform(ds, bank).save(os.path.join(out, "two_class_single.rkfm"))
    gr.transform(ds, bank, include_mpv=True).save(os.path.join(out, "two_class_mpv.rkfm"))
    gr.transform(ds, bank, precision="double").save(os.path.join(out, "two_class_double.rkfm"))
    gr.transform(ds64, bank).save(os.path.join(out, "random64_single.rkfm"))
    gr.transform(ds, bank).to_csv(os.path.join(out, "two_class_single.csv"))
    gr.transform(ds, bank, precision="double").to_csv(os.path.join(out, "two_class_double.csv"))


def make_ridge_models():
    """RKRM v1 model files written by the reference's RidgeModel.save
    (ridge.py:49-67): a one-vs-rest classifier and a regression model fitted
    on the reference features of the two-class cache."""
    from gridrocket import ridge as rr
    from gridrocket.data import load_cache

    out = os.path.join(HERE, "formats")
    ds = load_cache(os.path.join(out, "two_class.rkds"))
    bank = gr.generate_bank(40, 1, 6, gr.GenOptions(seed=5))
    feats = gr.transform(ds, bank)
    rr.fit(feats, ds.labels, alpha=0.5).save(os.path.join(out, "ridge_cls.rkrm"))
    rr.fit_regression(feats, np.arange(ds.values.shape[0], dtype=np.float64), alpha=2.0).save(
        os.path.join(out, "ridge_reg.rkrm"))


if __name__ == "__main__":
    if sys.argv[1:] == ["ridge_models"]:
        make_ridge_models()
    else:
        main()
