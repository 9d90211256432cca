"""Time the public numpy-in / numpy-out call (paper_2601_17091_b200.transform)
at config 2, split into its host stages, against the pinned-buffer C-ABI
path bench.py's e2e uses.

    python tools/public_api_timing.py [--n 100000] [--mode fast]
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

from paper_2601_17091_b200 import GenOptions, device_bank, generate_bank, synth_random, transform  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=100000)
ap.add_argument("--mode", default="fast")
args = ap.parse_args()
bank = generate_bank(1024, 1, 10000, GenOptions(seed=0))
values = synth_random(args.n, 1, 1024, seed=1).values
device_bank(bank, 0)
transform(values[:1000], bank, mode=args.mode)
for mode in ("fast", "exact"):
    for i in range(2):
        t = time.perf_counter()
        fm = transform(values, bank, mode=mode)
        dt = time.perf_counter() - t
        print(f"transform(mode={mode!r}): {args.n / dt:.0f} series/s ({dt:.3f} s)", flush=True)
        del fm
t = time.perf_counter()
ok = np.isfinite(values).all()
print(f"  np.isfinite scan: {time.perf_counter() - t:.3f} s", flush=True)
t = time.perf_counter()
out = np.empty((args.n, 20000), dtype=np.float32)
out[:, 0] = 0
out.fill(0)
print(f"  np.empty + first touch of the 8 GB output: {time.perf_counter() - t:.3f} s", flush=True)
