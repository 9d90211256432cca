"""Run a device-resident transform for ncu (one call, optional warm-up).

    python tools/profile_transform.py [--config config2] [--series N] [--mode fast] [--warmup 1]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from bench import CONFIGS  # noqa: E402
from paper_2601_17091_b200 import GenOptions, device_bank, generate_bank  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="config2")
ap.add_argument("--series", type=int, default=20000)
ap.add_argument("--kernels", type=int, default=None)
ap.add_argument("--mode", default="fast")
ap.add_argument("--warmup", type=int, default=1)
ap.add_argument("--fpk", type=int, default=2)
ap.add_argument("--precision", default="single")
args = ap.parse_args()
cfg = CONFIGS[args.config]
k = args.kernels or cfg["k"]
bank = generate_bank(cfg["l"], cfg["c"], k, GenOptions(seed=0))
db = device_bank(bank, 0)
dt = torch.float64 if args.precision == "double" else torch.float32
x = torch.randn((args.series, cfg["c"], cfg["l"]), device="cuda", dtype=dt)
out = torch.empty((args.series, args.fpk * k), device="cuda", dtype=dt)
s = torch.cuda.current_stream().cuda_stream
for _ in range(args.warmup + 1):
    db.transform_into(x.data_ptr(), args.series, out.data_ptr(), args.fpk * k, mode=args.mode, stream=s,
                      fpk=args.fpk, precision=args.precision)
torch.cuda.synchronize()
print("info", db.info)
