"""Parity checkers shared by the GPU tests and smoke().

exact mode: byte equality with the reference (oracle / golden fixtures).
fast mode:  the north-star tolerance (BASELINE.json): MAX within 1e-5
            relative (plus a 1e-6 absolute floor for maxima that are
            themselves within 1e-6 of zero), and PPV exact except for
            convolution outputs within 1e-6 of zero — every PPV mismatch is
            certified by a float64 recompute of that cell (oracle
            convolve_f64): |count_gpu - count_ref| <= #{t : |v64[t]| < 1e-6}.
"""

import numpy as np

MAX_RTOL = 1e-5
MAX_ATOL = 1e-6
# fast-mode MPV: a reordered float32 sum of positive terms (no cancellation)
MPV_RTOL = 1e-5
NEAR_ZERO = 1e-6


def check_fast(gpu, ref, values, bank, fpk=2):
    """Return a report dict; raise AssertionError if out of tolerance.

    fpk = 3 also checks MPV (fast mode sums the positive outputs per lane
    and then across the warp instead of in position order): within MPV_RTOL
    relative of the reference, widened for a cell whose count differs
    (certified above) by the share of the sum such near-zero outputs can
    move: |d mpv| <= mpv * |d count| / count + |d count| * NEAR_ZERO / count.
    """
    from oracle.oracle import convolve_f64

    gpu = np.asarray(gpu, dtype=np.float32)
    ref = np.asarray(ref, dtype=np.float32)
    assert gpu.shape == ref.shape
    gm, rm = gpu[:, 1::fpk].astype(np.float64), ref[:, 1::fpk].astype(np.float64)
    err = np.abs(gm - rm)
    bound = MAX_RTOL * np.abs(rm) + MAX_ATOL
    bad = err > bound
    assert not bad.any(), f"{int(bad.sum())} MAX cells out of tolerance; worst {err[bad].max()}"
    rel = err / np.maximum(np.abs(rm), 1e-30)
    l_out = bank.output_lengths()
    gp, rp = gpu[:, 0::fpk], ref[:, 0::fpk]
    mism = np.argwhere(gp != rp)
    x = np.asarray(values, dtype=np.float32)
    dcount = {}
    for i, k in mism:
        v = convolve_f64(x[i].astype(np.float64), bank, int(k))
        near = int(np.count_nonzero(np.abs(v) < NEAR_ZERO))
        cg = int(round(float(gp[i, k]) * l_out[k]))
        cr = int(round(float(rp[i, k]) * l_out[k]))
        assert abs(cg - cr) <= near, f"PPV cell ({i},{k}) differs by {cg - cr} with only {near} near-zero outputs"
        dcount[(int(i), int(k))] = (abs(cg - cr), max(1, min(cg, cr)))
    report = {"max_rel_err": float(rel.max()) if rel.size else 0.0, "ppv_mismatches": int(len(mism)),
              "cells": int(gp.size)}
    if fpk == 3:
        gv, rv = gpu[:, 2::3].astype(np.float64), ref[:, 2::3].astype(np.float64)
        bound = MPV_RTOL * np.abs(rv) + MAX_ATOL
        for (i, k), (dc, cnt) in dcount.items():
            bound[i, k] += abs(rv[i, k]) * dc / cnt + dc * NEAR_ZERO / cnt
        merr = np.abs(gv - rv)
        bad = merr > bound
        assert not bad.any(), f"{int(bad.sum())} MPV cells out of tolerance; worst {merr[bad].max()}"
        report["mpv_max_rel_err"] = float((merr / np.maximum(np.abs(rv), 1e-30)).max()) if rv.size else 0.0
    return report
