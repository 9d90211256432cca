#!/usr/bin/env python
"""ROCKET transform throughput on B200 — the driver's bench contract.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--mode fast|exact]
                    [--config config2|config4|config5] [--impl ours|reference]

A step is one transform of the rank's whole synthetic batch (BASELINE
configs[1]: 100,000 series x L=1024 with 10,000 kernels per GPU; under
torchrun every rank transforms its own 100,000-series shard — configs[2]'s
series-sharded layout with fixed per-GPU work, so "scaling": "weak").
`value` is device-resident throughput (inputs in HBM before the timed region,
CUDA events on the launching stream, max over ranks); `e2e` is the same
metric through the public C-ABI call with pinned host buffers (H2D of the
series and D2H of all features inside the timed region).
`--impl reference` times the reference algorithm on the host cores instead
(the pinned C restatement in oracle/, all threads, bounded samples).
"""

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

CONFIGS = {
    "config2": dict(n=100_000, c=1, l=1024, k=10_000,
                    workload="ROCKET transform, 10,000 kernels, 100,000 series x length 1,024 per GPU"),
    "config4": dict(n=20_000, c=1, l=16_384, k=10_000,
                    workload="ROCKET transform, 10,000 kernels, 20,000 series x length 16,384"),
    "config5": dict(n=50_000, c=3, l=2048, k=10_000,
                    workload="ROCKET transform, multivariate 3 channels, 50,000 series x length 2,048"),
    "uni2048": dict(n=50_000, c=1, l=2048, k=10_000,
                    workload="ROCKET transform, 10,000 kernels, 50,000 series x length 2,048"),
    "forda": dict(n=3_601, c=1, l=500, k=10_000,
                  workload="ROCKET transform, 10,000 kernels, 3,601 series x length 500 (FordA shape)"),
}
METRIC = "ROCKET transform series/sec (10k kernels, L=1024)"
FP32_PEAK_MEASURED = 74.0  # TFLOP/s, FFMA2 microbenchmark (profiles/r01_fp32_peak_microbench.jsonl)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--mode", choices=["fast", "exact"], default="fast")
    ap.add_argument("--config", choices=sorted(CONFIGS), default="config2")
    ap.add_argument("--kernels", type=int, default=None, help="override the kernel count (config5 sweep)")
    ap.add_argument("--series", type=int, default=None, help="override series per GPU")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-variants", action="store_true", help="skip the MPV / float64 throughput lines")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    return ap.parse_args()


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
        time.sleep(0.3)
        return self

    def __exit__(self, *exc):
        self.lines = []
        if self.proc is not None:
            time.sleep(0.2)
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
                out, _ = self.proc.communicate()
            self.lines = [ln for ln in out.splitlines() if ln.strip()]

    def summary(self):
        sm, mx, power, reasons = [], None, [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in getattr(self, "lines", []):
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 7:
                continue
            try:
                sm.append(float(f[0]))
                mx = float(f[1])
                power.append(float(f[2]))
            except ValueError:
                continue
            for nm, v in zip(names, f[3:7]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        load = [s for s, p in zip(sm, power) if p > 1.3 * min(power)] or sm
        return {"sm_mhz": float(np.median(load)), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "power_w_median": float(np.median(power)), "samples": len(sm)}


def nvml_energy_mj(index):
    try:
        import pynvml

        pynvml.nvmlInit()
        h = pynvml.nvmlDeviceGetHandleByIndex(index)
        return float(pynvml.nvmlDeviceGetTotalEnergyConsumption(h))
    except Exception:
        return None


def cpu_sample_rate(bank, cfg, seconds, seed=1):
    """Reference-algorithm throughput (series/s) on the host cores: the
    pinned C restatement (oracle/) with every host thread, on a bounded
    sample of the same workload sized to ~`seconds` of CPU work."""
    from oracle.oracle import oracle_transform
    from paper_2601_17091_b200 import synth_random

    threads = os.cpu_count() or 1
    probe = threads  # one series per thread, so the probe rate is the full-machine rate
    x = synth_random(probe, cfg["c"], cfg["l"], seed=seed).values
    oracle_transform(x, bank, nthreads=threads)  # warm (library load, thread start-up)
    t0 = time.perf_counter()
    oracle_transform(x, bank, nthreads=threads)
    t_probe = time.perf_counter() - t0
    m = int(max(threads, min(4096, probe * seconds / max(t_probe, 1e-3))))
    m = max(threads, (m // threads) * threads)
    x = synth_random(m, cfg["c"], cfg["l"], seed=seed).values
    t0 = time.perf_counter()
    oracle_transform(x, bank, nthreads=threads)
    dt = time.perf_counter() - t0
    return m / dt, m, dt, threads


def run_reference(args, cfg):
    """--impl reference: the reference algorithm on the host cores."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    import oracle.oracle as orc
    from paper_2601_17091_b200 import GenOptions, generate_bank, synth_random

    orc.build()
    bank = generate_bank(cfg["l"], cfg["c"], cfg["k"], GenOptions(seed=0))
    threads = os.cpu_count() or 1
    # one step = a bounded sample sized for ~2.5 s of CPU work
    rate, _, _, _ = cpu_sample_rate(bank, cfg, 2.5)
    m = max(threads, int(rate * 2.5 // threads) * threads)
    x = synth_random(m, cfg["c"], cfg["l"], seed=1).values
    for _ in range(args.warmup):
        orc.oracle_transform(x[:threads], bank, nthreads=threads)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        orc.oracle_transform(x, bank, nthreads=threads)
        times.append(time.perf_counter() - t0)
    total = sum(times)
    value = m * args.steps / total
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "series/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (synth_random seed 1; bank generate_bank seed 0)",
        "config": {"workload": cfg["workload"], "series_per_step": m, "l_series": cfg["l"],
                   "n_channels": cfg["c"], "n_kernels": cfg["k"], "parallelism": "cpu threads"},
        "cpu_baseline": {"value": value, "unit": "series/s", "cores": threads, "kind": "port",
                         "sample": f"{m} series per step of the {cfg['workload']} workload"},
        "e2e": {"value": value, "unit": "series/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    cfg = dict(CONFIGS[args.config])
    if args.kernels:
        cfg["k"] = args.kernels
    if args.series:
        cfg["n"] = args.series
    if args.impl == "reference":
        return run_reference(args, cfg)

    import torch
    import torch.distributed as dist

    from paper_2601_17091_b200 import GenOptions, device_bank, generate_bank, synth_random

    rank, world, local = dist_env()
    # one process per GPU; the modulo only matters for a logic check of the
    # multi-rank path on a box with fewer GPUs than ranks
    local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    if world > 1:
        backend = os.environ.get("RK_BENCH_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)

    bank = generate_bank(cfg["l"], cfg["c"], cfg["k"], GenOptions(seed=0))
    db = device_bank(bank, local)
    info = db.info
    n = cfg["n"]
    fpk = 2
    # synthetic per-rank shard (seed 1 + rank), float32 like synth_random
    x_host = torch.from_numpy(synth_random(n, cfg["c"], cfg["l"], seed=1 + rank).values).pin_memory()
    x_dev = x_host.cuda()
    out_dev = torch.empty((n, bank.count * fpk), device="cuda", dtype=torch.float32)
    stream = torch.cuda.Stream()
    sptr = stream.cuda_stream

    def step(mode, xp, op):
        return db.transform_into(xp, n, op, bank.count * fpk, mode=mode, stream=sptr)

    def barrier():
        if world > 1:
            dist.barrier()

    def timed(mode):
        for _ in range(args.warmup):
            step(mode, x_dev.data_ptr(), out_dev.data_ptr())
        torch.cuda.synchronize()
        barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            step(mode, x_dev.data_ptr(), out_dev.data_ptr())
        e1.record(stream)
        torch.cuda.synchronize()
        barrier()
        ms = e0.elapsed_time(e1)
        t = torch.tensor([ms], device="cuda", dtype=torch.float64)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # ---- headline: device-resident, selected mode -------------------------
    e_before = nvml_energy_mj(local)
    with ClockSampler(local) as clk:
        ms_total = timed(args.mode)
    e_after = nvml_energy_mj(local)
    ms_step = ms_total / args.steps
    total_series = n * world * args.steps
    value = total_series / (ms_total / 1e3)
    flops_series = info["useful_flops_per_series"]
    achieved_tflops = flops_series * n / (ms_step / 1e3) / 1e12

    # ---- the other mode, same protocol -----------------------------------
    other = "exact" if args.mode == "fast" else "fast"
    ms_other = timed(other)

    # ---- the other feature sets, device-resident, on a 20k-series slice ----
    variants = None
    if not args.no_variants:
        variants = {}
        nv = min(n, 20000)
        for name, fpk_v, prec, mode_v in (("mpv_fast", 3, "single", "fast"), ("mpv_exact", 3, "single", "exact"),
                                          ("double", 2, "double", "exact")):
            dt = torch.float64 if prec == "double" else torch.float32
            xv = x_dev[:nv].to(dt).contiguous()
            ov = torch.empty((nv, bank.count * fpk_v), device="cuda", dtype=dt)
            db.transform_into(xv.data_ptr(), nv, ov.data_ptr(), bank.count * fpk_v, mode=mode_v, fpk=fpk_v,
                              precision=prec, stream=sptr)
            torch.cuda.synchronize()
            ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            ev0.record(stream)
            db.transform_into(xv.data_ptr(), nv, ov.data_ptr(), bank.count * fpk_v, mode=mode_v, fpk=fpk_v,
                              precision=prec, stream=sptr)
            ev1.record(stream)
            torch.cuda.synchronize()
            variants[name] = {"value": nv / (ev0.elapsed_time(ev1) / 1e3), "unit": "series/s", "series": nv,
                              "fpk": fpk_v, "precision": prec, "mode": mode_v}
            del xv, ov

    # ---- e2e through the public C-ABI call with pinned host buffers --------
    e2e = None
    if not args.no_e2e:
        out_host = torch.empty((n, bank.count * fpk), dtype=torch.float32).pin_memory()
        for _ in range(1):
            db.transform_into(x_host.data_ptr(), n, out_host.data_ptr(), bank.count * fpk, mode=args.mode)
        barrier()
        with ClockSampler(local) as clk_e2e:
            t0 = time.perf_counter()
            for _ in range(args.steps):
                db.transform_into(x_host.data_ptr(), n, out_host.data_ptr(), bank.count * fpk, mode=args.mode)
                _ = float(out_host[n - 1, 1])  # the step's result read on the host
            dt = time.perf_counter() - t0
        t = torch.tensor([dt], device="cuda", dtype=torch.float64)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dt = float(t.item())
        e2e = {"value": total_series / dt, "unit": "series/s",
               "h2d_bytes_per_step": int(x_host.numel() * 4),
               "d2h_bytes_per_step": int(out_host.numel() * 4),
               "ms_per_step": 1e3 * dt / args.steps,
               "clocks": clk_e2e.summary(),
               "path": "DeviceBank.transform_into -> rk_transform (host pinned x/out, pipelined H2D/kernel/D2H)"}
        del out_host

    # ---- CPU baseline on rank 0 at N=1 -------------------------------------
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        import oracle.oracle as orc

        orc.build()
        rate, m, dt, threads = cpu_sample_rate(bank, cfg, args.cpu_seconds)
        cpu = {"value": rate, "unit": "series/s", "cores": threads, "kind": "port",
               "sample": f"{m} series of the same workload (synth_random seed 1), {dt:.1f} s, "
                         "oracle/rocket_oracle.c restating engine._run_batch, pthreads"}

    energy = None
    if e_before is not None and e_after is not None:
        joules = (e_after - e_before) / 1e3
        energy = {"joules_rank0": joules,
                  "features_per_joule": n * bank.count * fpk * args.steps / joules if joules > 0 else None}

    traffic = None
    prof = os.path.join(ROOT, "profiles", f"ncu_summary_{args.config}.json")
    if os.path.exists(prof):
        try:
            with open(prof) as f:
                traffic = json.load(f).get("dram_bytes_per_series")
            if traffic is not None:
                traffic = traffic * n
        except Exception:
            traffic = None

    if rank == 0:
        line = {
            "metric": METRIC,
            "value": value,
            "unit": "series/s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": ms_step,
            "higher_is_better": True,
            "scaling": "weak",
            "vs_baseline": None,
            "dtype": "f32",
            "mode": args.mode,
            "data": "synthetic: synth_random(seed=1+rank) float32 series, generate_bank(seed=0) kernels",
            "config": {"workload": cfg["workload"], "series_per_gpu": n, "l_series": cfg["l"],
                       "n_channels": cfg["c"], "n_kernels": bank.count, "parallelism": f"series-sharded x{world}",
                       "l2": "inputs (%.0f MB/GPU) and outputs (%.1f GB/GPU) exceed the 126 MB L2"
                             % (x_host.numel() * 4 / 1e6, n * bank.count * fpk * 4 / 1e9)},
            "roofline": {"bound": "fp32", "achieved": achieved_tflops, "peak": FP32_PEAK_MEASURED,
                         "unit": "TFLOP/s", "frac": achieved_tflops / FP32_PEAK_MEASURED, "traffic": traffic,
                         "flops_per_series": flops_series,
                         "algorithmic_bytes": (4 * cfg["c"] * cfg["l"] + 4 * fpk * bank.count) * n,
                         "hbm_GBps": (traffic / (ms_step / 1e3) / 1e9) if traffic else None,
                         "traffic_source": "profiles/ncu_summary_%s.json (ncu dram bytes of one transform, "
                                           "scaled to this step's series)" % args.config if traffic else None,
                         "peak_source": "measured FFMA2 microbenchmark (profiles/r01_fp32_peak_microbench.jsonl); "
                                        "MEASURED_PEAKS.json has no FP32 entry",
                         "kernel": ("rocket_class_kernel" if info["path"] == 0 else "rocket_wide_kernel")
                                   + f" x {info['n_launches']} launches (one transform; DESIGN.md §4)"},
            "other_mode": {"mode": other, "ms_per_step": ms_other / args.steps,
                           "value": total_series / (ms_other / 1e3),
                           "achieved_tflops": flops_series * n / (ms_other / args.steps / 1e3) / 1e12},
            "e2e": e2e,
            "variants": variants,
            "cpu_baseline": cpu,
            "clocks": clk.summary(),
            "energy": energy,
            "gpu_launches": int(info["n_launches"]) * args.steps,
            "bank": {"groups": info["n_groups"], "chunks": info["n_chunks"], "launches_per_step": info["n_launches"],
                     "smem_bytes": info["smem_bytes"], "path": {0: "class", 1: "wide", 2: "wide (series in global memory)"}[info["path"]],
                     "ctas_per_sm": info["ctas_per_sm"]},
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
