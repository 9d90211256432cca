"""Diagnose the host-buffer (e2e) path: raw copy bandwidths vs transform_into."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2601_17091_b200 import GenOptions, device_bank, generate_bank, synth_random

n = int(sys.argv[1]) if len(sys.argv) > 1 else 100000
bank = generate_bank(1024, 1, 10000, GenOptions(seed=0))
db = device_bank(bank, 0)
xh = torch.from_numpy(synth_random(n, 1, 1024, seed=1).values).pin_memory()
oh = torch.empty((n, 20000), dtype=torch.float32).pin_memory()
od = torch.empty((n, 20000), device="cuda")
xd = xh.cuda()
torch.cuda.synchronize()
for _ in range(2):
    t = time.perf_counter(); oh.copy_(od, non_blocking=True); torch.cuda.synchronize(); dt = time.perf_counter() - t
    print("D2H %.1f GB at %.1f GB/s" % (oh.numel() * 4 / 1e9, oh.numel() * 4 / dt / 1e9))
    t = time.perf_counter(); xd.copy_(xh, non_blocking=True); torch.cuda.synchronize(); dt = time.perf_counter() - t
    print("H2D %.2f GB at %.1f GB/s" % (xh.numel() * 4 / 1e9, xh.numel() * 4 / dt / 1e9))
s = torch.cuda.Stream()
for mode in ("fast", "fast", "fast"):
    t = time.perf_counter(); db.transform_into(xd.data_ptr(), n, od.data_ptr(), 20000, mode=mode, stream=s.cuda_stream); dt = time.perf_counter() - t
    print("device %s %.1f ms" % (mode, dt * 1e3))
for mode in ("fast", "fast", "fast"):
    t = time.perf_counter(); db.transform_into(xh.data_ptr(), n, oh.data_ptr(), 20000, mode=mode); dt = time.perf_counter() - t
    print("host %s %.1f ms" % (mode, dt * 1e3))
