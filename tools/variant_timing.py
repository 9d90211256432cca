"""Device-resident throughput of the cell-kernel variants (exact MPV,
float64 in both modes' cell path) at a config's shape, optionally A/B with
an environment switch set inside the process.

    python tools/variant_timing.py [--config config2] [--series 20000]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from bench import CONFIGS  # noqa: E402
from paper_2601_17091_b200 import GenOptions, device_bank, generate_bank  # noqa: E402
from paper_2601_17091_b200.engine import DeviceBank  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="config2")
ap.add_argument("--series", type=int, default=20000)
args = ap.parse_args()
cfg = CONFIGS[args.config]
bank = generate_bank(cfg["l"], cfg["c"], cfg["k"], GenOptions(seed=0))
n = args.series
x32 = torch.randn((n, cfg["c"], cfg["l"]), device="cuda")
x64 = x32.double()


def run(db, mode, fpk, precision):
    x = x64 if precision == "double" else x32
    out = torch.empty((n, bank.count * fpk), device="cuda", dtype=x.dtype)
    s = torch.cuda.current_stream()
    db.transform_into(x.data_ptr(), n, out.data_ptr(), out.shape[1], mode=mode, fpk=fpk, precision=precision,
                      stream=s.cuda_stream)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    db.transform_into(x.data_ptr(), n, out.data_ptr(), out.shape[1], mode=mode, fpk=fpk, precision=precision,
                      stream=s.cuda_stream)
    e1.record(s)
    torch.cuda.synchronize()
    return n / (e0.elapsed_time(e1) / 1e3), out


for label, env in (("paired", None), ("cellrow", "RK_NO_CELLPAIR")):
    if env:
        os.environ[env] = "1"
    db = DeviceBank(bank, 0)
    r1, a = run(db, "exact", 3, "single")
    r2, b = run(db, "exact", 2, "double")
    print(f"{args.config} {label}: exact MPV {r1:.0f} series/s, float64 {r2:.0f} series/s", flush=True)
    if env:
        del os.environ[env]
        assert torch.equal(a, ref_a) and torch.equal(b, ref_b), "paired and cellrow kernels differ"
        print("bytes equal between the two kernels")
    else:
        ref_a, ref_b = a, b
    db.close()
