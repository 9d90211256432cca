"""Parity checkers shared by the GPU tests and smoke() — TEST INFRASTRUCTURE
ONLY (imported by tests/ and __graft_entry__.smoke(), never by the product).

exact mode: byte equality with the reference (oracle / golden fixtures).

fast mode: the north-star tolerance (BASELINE.json) — "MAX within 1e-5
relative and PPV exact except for convolution outputs within 1e-6 of zero" —
checked cell by cell against the reference's float32 features:

* MAX: |g - r| <= 1e-5 |r|.  The 1e-6 absolute floor applies only to a
  reference maximum that is itself within 1e-6 of zero.
* Every MAX cell outside that rule must be *certified* by a float64
  recomputation from the same float32 operands (oracle.cell_cert): both the
  GPU value and the reference value lie within the float32 forward-error
  bound e = gamma(m+1) * max_t (|b| + sum |w x|) of the float64 maximum
  (Higham eq. 3.5; any summation order, with or without FMA).  Such a cell
  is one whose output cancels so far that float32 itself cannot resolve it
  to 1e-5 — the reference's own float32 answer is that far from the truth
  too.  The test data are never rescaled to avoid these cells.
* PPV: every mismatching cell's GPU count must equal the float64 count up to
  the outputs whose sign float32 cannot decide (|v64| <= max(1e-6, e_t));
  the report separates flips explained by the 1e-6 band alone.
* MPV (fpk = 3): within 1e-5 relative of the reference (widened by the
  certified count difference), else certified against the float64 positive
  mean with the same per-output bounds plus the summation bound of the
  positive terms.
"""

import numpy as np

MAX_RTOL = 1e-5
NEAR_ZERO = 1e-6
MPV_RTOL = 1e-5
U32 = 2.0 ** -24


def _gamma(n):
    n = np.asarray(n, dtype=np.float64)
    return n * U32 / (1.0 - n * U32)


def check_fast(gpu, ref, values, bank, fpk=2):
    """Return a report dict; raise AssertionError if any cell is out of
    tolerance and not certified."""
    from oracle.oracle import cell_cert

    gpu = np.asarray(gpu, dtype=np.float32)
    ref = np.asarray(ref, dtype=np.float32)
    assert gpu.shape == ref.shape, (gpu.shape, ref.shape)
    x = np.asarray(getattr(values, "values", values), dtype=np.float32)
    l_out = bank.output_lengths()

    # ---- MAX ---------------------------------------------------------------
    gm, rm = gpu[:, 1::fpk].astype(np.float64), ref[:, 1::fpk].astype(np.float64)
    assert np.isfinite(gm).all(), "non-finite MAX from the GPU"
    err = np.abs(gm - rm)
    ok = err <= MAX_RTOL * np.abs(rm)
    ok |= (np.abs(rm) < NEAR_ZERO) & (err <= NEAR_ZERO)
    cand = np.argwhere(~ok)
    max_cert = 0
    if len(cand):
        c = cell_cert(x, bank, cand[:, 0], cand[:, 1])
        g_in = np.abs(gm[cand[:, 0], cand[:, 1]] - c["max64"]) <= c["maxerr"]
        r_in = np.abs(rm[cand[:, 0], cand[:, 1]] - c["max64"]) <= c["maxerr"]
        bad = ~(g_in & r_in)
        if bad.any():
            i, k = cand[bad][0]
            j = int(np.argmax(bad))
            raise AssertionError(
                f"{int(bad.sum())} MAX cells out of tolerance and not certified; first ({i},{k}): "
                f"gpu {gm[i, k]!r} ref {rm[i, k]!r} f64 {c['max64'][j]!r} bound {c['maxerr'][j]!r}")
        max_cert = len(cand)
    rel = err / np.maximum(np.abs(rm), 1e-30)
    rel_unc = np.where(ok, rel, 0.0)

    # ---- PPV ---------------------------------------------------------------
    gp, rp = gpu[:, 0::fpk], ref[:, 0::fpk]
    mism = np.argwhere(gp != rp)
    ppv_band = ppv_fp32 = 0
    cg = cr = None
    cert = None
    if len(mism):
        cert = cell_cert(x, bank, mism[:, 0], mism[:, 1])
        lo = l_out[mism[:, 1]]
        cg = np.rint(gp[mism[:, 0], mism[:, 1]].astype(np.float64) * lo).astype(np.int64)
        cr = np.rint(rp[mism[:, 0], mism[:, 1]].astype(np.float64) * lo).astype(np.int64)
        dg = np.abs(cg - cert["pos"])
        dr = np.abs(cr - cert["pos"])
        bad = (dg > cert["unsure"]) | (dr > cert["unsure"])
        if bad.any():
            j = int(np.argmax(bad))
            i, k = mism[j]
            raise AssertionError(
                f"{int(bad.sum())} PPV cells differ beyond the undecided outputs; first ({i},{k}): gpu count "
                f"{cg[j]} ref {cr[j]} f64 {cert['pos'][j]} undecided {cert['unsure'][j]} "
                f"(within 1e-6: {cert['near'][j]})")
        within_band = np.abs(cg - cr) <= cert["near"]
        ppv_band = int(within_band.sum())
        ppv_fp32 = int((~within_band).sum())

    report = {"cells": int(gm.size), "max_rel_err": float(rel.max()) if rel.size else 0.0,
              "max_rel_err_uncertified": float(rel_unc.max()) if rel.size else 0.0,
              "max_certified_cells": int(max_cert), "ppv_mismatches": int(len(mism)),
              "ppv_flips_within_1e-6": ppv_band, "ppv_flips_fp32_undecided": ppv_fp32}
    assert report["max_rel_err_uncertified"] <= MAX_RTOL

    # ---- MPV ---------------------------------------------------------------
    if fpk == 3:
        gv, rv = gpu[:, 2::3].astype(np.float64), ref[:, 2::3].astype(np.float64)
        bound = MPV_RTOL * np.abs(rv)
        if len(mism):
            dc = np.abs(cg - cr)
            cnt = np.maximum(1, np.minimum(cg, cr))
            bound[mism[:, 0], mism[:, 1]] += np.abs(rv[mism[:, 0], mism[:, 1]]) * dc / cnt + dc * NEAR_ZERO / cnt
        merr = np.abs(gv - rv)
        ok = merr <= bound
        cand = np.argwhere(~ok)
        mpv_cert = 0
        if len(cand):
            c = cell_cert(x, bank, cand[:, 0], cand[:, 1])
            lo = l_out[cand[:, 1]]
            gcount = np.rint(gp[cand[:, 0], cand[:, 1]].astype(np.float64) * lo)
            npos = c["pos"].astype(np.float64)
            mpv64 = np.where(npos > 0, c["psum64"] / np.maximum(npos, 1), 0.0)
            sum_err = c["psumerr"] + _gamma(np.maximum(npos + c["unsure"], 1)) * (c["psum64"] + c["psumerr"])
            gb = np.where(gcount > 0, sum_err / np.maximum(gcount, 1) + mpv64 * np.abs(npos - gcount)
                          / np.maximum(gcount, 1), c["psum64"] + c["psumerr"])
            bad = np.abs(gv[cand[:, 0], cand[:, 1]] - mpv64) > gb
            if bad.any():
                j = int(np.argmax(bad))
                i, k = cand[j]
                raise AssertionError(
                    f"{int(bad.sum())} MPV cells out of tolerance and not certified; first ({i},{k}): gpu "
                    f"{gv[i, k]!r} ref {rv[i, k]!r} f64 {mpv64[j]!r} bound {gb[j]!r}")
            mpv_cert = len(cand)
        report["mpv_max_rel_err"] = float((merr / np.maximum(np.abs(rv), 1e-30)).max()) if rv.size else 0.0
        report["mpv_certified_cells"] = int(mpv_cert)
    return report
