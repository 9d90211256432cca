"""The reference's own CPU transform (gridrocket.transform, numba, from
/root/reference in this container) against the C port used as the bench's
reference arm (oracle/rocket_oracle.c), on the same host, same sample:
shows the port is at least as fast as the reference, so GPU / port ratios
understate GPU / reference.

    NUMBA_CACHE_DIR=/tmp/numba_cache python tools/cpu_reference_vs_port.py [--n 200] [--out JSON]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=200)
    ap.add_argument("--out")
    args = ap.parse_args()
    import gridrocket as gr
    import numba

    from oracle.oracle import build, oracle_transform
    from paper_2601_17091_b200 import GenOptions, generate_bank, synth_random

    build()
    bank_ref = gr.generate_bank(1024, 1, 10000, gr.GenOptions(seed=0))
    bank = generate_bank(1024, 1, 10000, GenOptions(seed=0))
    values = synth_random(args.n, 1, 1024, seed=1).values
    gr.transform(values[:2], bank_ref)  # numba compile
    t = time.perf_counter()
    ref = gr.transform(values, bank_ref).values
    t_ref = time.perf_counter() - t
    oracle_transform(values[:2], bank)
    t = time.perf_counter()
    port = oracle_transform(values, bank)
    t_port = time.perf_counter() - t
    res = {"n_series": args.n, "workload": "10k kernels, L=1024 (config 2 bank and series)",
           "cpu_count": os.cpu_count(), "numba_threads": numba.get_num_threads(),
           "numba_threading_layer": numba.threading_layer(),
           "reference_series_per_s": args.n / t_ref, "port_series_per_s": args.n / t_port,
           "port_over_reference": t_ref / t_port, "identical_bytes": bool(ref.tobytes() == port.tobytes())}
    print(json.dumps(res))
    if args.out:
        with open(args.out, "w") as f:
            json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
