"""Throughput for series longer than shared memory holds (GMEM path):
single-channel L = 32k / 65k and an EigenWorms-shaped set (6 x 17,984).

    python tools/long_series_timing.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2601_17091_b200 import GenOptions, device_bank, generate_bank  # noqa: E402
from paper_2601_17091_b200.engine import useful_flops_per_series  # noqa: E402

for C, L, n in ((1, 16384, 4000), (1, 32768, 2000), (1, 65536, 1000), (6, 17984, 1000)):
    bank = generate_bank(L, C, 10000, GenOptions(seed=0))
    db = device_bank(bank, 0)
    x = torch.randn((n, C, L), device="cuda")
    out = torch.empty((n, 20000), device="cuda")
    s = torch.cuda.current_stream()
    for mode in ("fast", "exact"):
        db.transform_into(x.data_ptr(), n, out.data_ptr(), 20000, mode=mode, stream=s.cuda_stream)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        db.transform_into(x.data_ptr(), n, out.data_ptr(), 20000, mode=mode, stream=s.cuda_stream)
        e1.record(s)
        torch.cuda.synchronize()
        dt = e0.elapsed_time(e1) / 1e3
        tf = useful_flops_per_series(bank) * n / dt / 1e12
        path = {0: "class", 1: "wide/smem", 2: "wide/global"}[db.info["path"]]
        print(f"C={C} L={L} {mode}: {n / dt:.0f} series/s, {tf:.1f} TFLOP/s, path={path}", flush=True)
