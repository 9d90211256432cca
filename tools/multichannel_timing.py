"""Throughput of multichannel banks beyond config 5 (kernels reading >= 3
channels run the class kernel, not the wide kernel).

    python tools/multichannel_timing.py
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2601_17091_b200 import GenOptions, device_bank, generate_bank  # noqa: E402
from paper_2601_17091_b200.engine import useful_flops_per_series  # noqa: E402

for C, L, n in ((3, 2048, 20000), (4, 1024, 20000), (8, 512, 20000), (16, 256, 20000)):
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
        print(f"C={C} L={L} {mode}: {n / dt:.0f} series/s, {tf:.1f} TFLOP/s, path={'wide' if db.info['path'] == 1 else 'class'}",
              flush=True)
