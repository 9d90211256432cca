"""Throughput of the cell-kernel paths (MPV, precision double) on config-2-shaped data."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2601_17091_b200 import GenOptions, device_bank, generate_bank

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4000
bank = generate_bank(1024, 1, 10000, GenOptions(seed=0))
db = device_bank(bank, 0)
s = torch.cuda.Stream()
for prec, fpk, mode in (("single", 3, "exact"), ("single", 3, "fast"), ("double", 2, "exact"), ("double", 3, "exact")):
    dt = torch.float64 if prec == "double" else torch.float32
    x = torch.randn((n, 1, 1024), device="cuda", dtype=dt)
    out = torch.empty((n, 10000 * fpk), device="cuda", dtype=dt)
    for i in range(3):
        torch.cuda.synchronize(); t = time.perf_counter()
        db.transform_into(x.data_ptr(), n, out.data_ptr(), 10000 * fpk, fpk=fpk, precision=prec, mode=mode, stream=s.cuda_stream)
        torch.cuda.synchronize(); el = time.perf_counter() - t
    print(f"{prec} fpk={fpk} {mode}: {n / el:.0f} series/s ({el * 1e3:.1f} ms for {n})", flush=True)
