"""Host bank generation: the reference's generate_bank (numpy draws, run
from /root/reference in this container) vs rk_generate_bank (SURVEY.md §8
f4), with a bit-identity check of every field.

    NUMBA_CACHE_DIR=/tmp/numba_cache python tools/bank_gen_timing.py [--out JSON]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import gridrocket as gr  # noqa: E402

from paper_2601_17091_b200.kernels import GenOptions, generate_bank  # noqa: E402

FIELDS = ("lengths", "weights", "biases", "dilations", "paddings", "channel_counts", "channel_indices")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out")
    args = ap.parse_args()
    rows = []
    for l_series, n_channels, count in ((1024, 1, 10000), (1024, 1, 100000), (2048, 3, 10000), (2048, 3, 100000),
                                        (16384, 1, 10000)):
        t0 = time.perf_counter()
        ref = gr.generate_bank(l_series, n_channels, count, gr.GenOptions(seed=0))
        t1 = time.perf_counter()
        nat = generate_bank(l_series, n_channels, count, GenOptions(seed=0), native=True)
        t2 = time.perf_counter()
        same = all(getattr(ref, f).tobytes() == getattr(nat, f).tobytes() for f in FIELDS)
        rows.append({"l_series": l_series, "n_channels": n_channels, "count": count, "reference_s": t1 - t0,
                     "native_s": t2 - t1, "speedup": (t1 - t0) / (t2 - t1), "bit_identical": same})
        print(json.dumps(rows[-1]))
    if args.out:
        with open(args.out, "w") as f:
            json.dump({"host": os.uname().nodename, "cpu_count": os.cpu_count(), "rows": rows}, f, indent=1)


if __name__ == "__main__":
    main()
