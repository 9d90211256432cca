"""Diagnose per-step host/GPU time of the device-resident transform."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2601_17091_b200 import GenOptions, device_bank, generate_bank, synth_random

n = int(sys.argv[1]) if len(sys.argv) > 1 else 100000
bank = generate_bank(1024, 1, 10000, GenOptions(seed=0))
db = device_bank(bank, 0)
x = torch.from_numpy(synth_random(n, 1, 1024, seed=1).values).cuda()
out = torch.empty((n, 20000), device="cuda")
stream = torch.cuda.Stream()
for mode in ("fast", "fast", "exact"):
    for i in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        e0.record(stream)
        db.transform_into(x.data_ptr(), n, out.data_ptr(), 20000, mode=mode, stream=stream.cuda_stream)
        e1.record(stream)
        t1 = time.perf_counter()
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        print(mode, "call %.1f ms, gpu %.1f ms, wall %.1f ms" % ((t1 - t0) * 1e3, e0.elapsed_time(e1), (t2 - t0) * 1e3), flush=True)
