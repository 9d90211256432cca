"""File-to-file transform throughput: RKDS cache ->
RKFM feature file through rk_transform_stream, against the reference's
sequence (load the cache, transform in memory, FeatureMatrix.save) run with
this repo's GPU transform, and against the disk's own write speed.

    python tools/file_pipeline.py [--n 20000] [--dir /tmp] [--out JSON]
"""

import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2601_17091_b200 import engine  # noqa: E402
from paper_2601_17091_b200.data import load_cache, save_cache, synth_random  # noqa: E402
from paper_2601_17091_b200.kernels import GenOptions, generate_bank  # noqa: E402
from paper_2601_17091_b200.stream import transform_file  # noqa: E402


def drop(path):
    if os.path.exists(path):
        os.remove(path)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=20000)
    ap.add_argument("--dir", default="/tmp")
    ap.add_argument("--mode", default="fast")
    ap.add_argument("--out")
    args = ap.parse_args()
    bank = generate_bank(1024, 1, 10000, GenOptions(seed=0))
    src = os.path.join(args.dir, "rk_pipe_in.rkds")
    dst = os.path.join(args.dir, "rk_pipe_out.rkfm")
    save_cache(synth_random(args.n, 1, 1024, seed=1), src)
    out_bytes = args.n * bank.count * 2 * 4
    res = {"n_series": args.n, "in_bytes": os.path.getsize(src), "out_bytes": out_bytes, "mode": args.mode,
           "dir": args.dir}
    # warm: bank upload, pinned ring, kernels
    transform_file(src, bank, dst, mode=args.mode, batch_rows=4096)
    drop(dst)

    # raw disk write of the same byte count (pinned-free numpy buffer)
    buf = np.zeros(256 << 20, dtype=np.uint8)
    t = time.perf_counter()
    with open(dst, "wb") as f:
        left = out_bytes
        while left > 0:
            f.write(buf[: min(left, buf.size)])
            left -= min(left, buf.size)
        f.flush()
        os.fsync(f.fileno())
    res["disk_write_GBps"] = out_bytes / (time.perf_counter() - t) / 1e9
    drop(dst)

    for label, sync in (("stream", False), ("stream_fsync", True)):
        t = time.perf_counter()
        transform_file(src, bank, dst, mode=args.mode)
        if sync:
            fd = os.open(dst, os.O_RDONLY)
            os.fsync(fd)
            os.close(fd)
        dt = time.perf_counter() - t
        res[f"{label}_s"] = dt
        res[f"{label}_series_per_s"] = args.n / dt
        res[f"{label}_out_GBps"] = out_bytes / dt / 1e9
        drop(dst)

    # the reference's sequence: load_cache -> transform -> save
    t = time.perf_counter()
    ds = load_cache(src)
    fm = engine.transform(ds, bank, mode=args.mode)
    t1 = time.perf_counter()
    fm.save(dst)
    dt = time.perf_counter() - t
    res["in_memory_then_save_s"] = dt
    res["in_memory_transform_s"] = t1 - t
    res["in_memory_series_per_s"] = args.n / dt
    drop(dst)
    drop(src)
    print(json.dumps(res))
    if args.out:
        with open(args.out, "w") as f:
            json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
