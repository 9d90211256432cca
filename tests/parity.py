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
NEAR_ZERO = 1e-6


def check_fast(gpu, ref, values, bank):
    """Return a report dict; raise AssertionError if out of tolerance."""
    from oracle.oracle import convolve_f64

    gpu = np.asarray(gpu, dtype=np.float32)
    ref = np.asarray(ref, dtype=np.float32)
    assert gpu.shape == ref.shape
    gm, rm = gpu[:, 1::2].astype(np.float64), ref[:, 1::2].astype(np.float64)
    err = np.abs(gm - rm)
    bound = MAX_RTOL * np.abs(rm) + MAX_ATOL
    bad = err > bound
    assert not bad.any(), f"{int(bad.sum())} MAX cells out of tolerance; worst {err[bad].max()}"
    rel = err / np.maximum(np.abs(rm), 1e-30)
    l_out = bank.output_lengths()
    gp, rp = gpu[:, 0::2], ref[:, 0::2]
    mism = np.argwhere(gp != rp)
    x = np.asarray(values, dtype=np.float32)
    for i, k in mism:
        v = convolve_f64(x[i].astype(np.float64), bank, int(k))
        near = int(np.count_nonzero(np.abs(v) < NEAR_ZERO))
        cg = int(round(float(gp[i, k]) * l_out[k]))
        cr = int(round(float(rp[i, k]) * l_out[k]))
        assert abs(cg - cr) <= near, f"PPV cell ({i},{k}) differs by {cg - cr} with only {near} near-zero outputs"
    return {"max_rel_err": float(rel.max()) if rel.size else 0.0, "ppv_mismatches": int(len(mism)),
            "cells": int(gp.size)}
