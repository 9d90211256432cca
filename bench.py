#!/usr/bin/env python
"""ROCKET transform throughput on B200 — the driver's bench contract.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--mode fast|exact]
                    [--config config2|config3|config4|config5|forda|uni2048]
                    [--impl ours|reference]

A step is one transform of the rank's whole synthetic batch.  Default
(BASELINE configs[1]): 100,000 series x L=1024 with 10,000 kernels per GPU;
under torchrun every rank transforms its own 100,000-series shard
("scaling": "weak").  `--config config3` is BASELINE configs[2]: 1,000,000
series split across the ranks by plan_shards (engine.py:123-134), "scaling":
"strong".  `value` is device-resident throughput (inputs in HBM before the
timed region, CUDA events on the launching stream, max over ranks); `e2e` is
the same metric through the public C-ABI call with pinned host buffers (H2D
of the series and D2H of all features inside the timed region);
`e2e_public` times the reference-facing numpy `transform()` (pageable
buffers) in both modes.  Energy is the NVML counter bracketing the timed
steps only, summed over ranks; the paper's per-watt metric (nominal power,
reference bench.py:62-70) is reported beside it.
`--impl reference` times the reference algorithm on the host cores instead
(the pinned C restatement in oracle/, all threads, bounded samples).
"""

import argparse
import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

CONFIGS = {
    "config1": dict(n=3_601, c=1, l=500, k=10_000, scaling="weak",
                    workload="ROCKET transform + ridge fit/predict, 10,000 kernels, 3,601 labelled series x "
                             "length 500 (FordA shape, synth_two_class)"),
    "config2": dict(n=100_000, c=1, l=1024, k=10_000, scaling="weak",
                    workload="ROCKET transform, 10,000 kernels, 100,000 series x length 1,024 per GPU"),
    "config3": dict(n=1_000_000, c=1, l=1024, k=10_000, scaling="strong",
                    workload="ROCKET transform, 10,000 kernels, 1,000,000 series x length 1,024 "
                             "series-sharded across the GPUs (plan_shards)"),
    "config4": dict(n=20_000, c=1, l=16_384, k=10_000, scaling="weak",
                    workload="ROCKET transform, 10,000 kernels, 20,000 series x length 16,384"),
    "config5": dict(n=50_000, c=3, l=2048, k=10_000, scaling="weak",
                    workload="ROCKET transform, multivariate 3 channels, 50,000 series x length 2,048"),
    "uni2048": dict(n=50_000, c=1, l=2048, k=10_000, scaling="weak",
                    workload="ROCKET transform, 10,000 kernels, 50,000 series x length 2,048"),
    "forda": dict(n=3_601, c=1, l=500, k=10_000, scaling="weak",
                  workload="ROCKET transform, 10,000 kernels, 3,601 series x length 500 (FordA shape)"),
}
METRIC = "ROCKET transform series/sec (10k kernels, L=1024)"
FP32_PEAK_MEASURED = 74.0  # TFLOP/s, FFMA2 microbenchmark (profiles/r01_fp32_peak_microbench.jsonl)
GPU_NOMINAL_W = 1000.0     # B200 board power limit (nvidia-smi power.limit), the paper's "nominal power"
E2E_BLOCK = 100_000        # config3 e2e: rows per public call (one reusable pinned output block)

# Nominal package power and hardware threads per package of host CPUs seen on
# B200 boxes (vendor TDP figures), for the paper's per-watt arithmetic.
CPU_TDP = {
    "Intel(R) Xeon(R) Platinum 8570": (350.0, 112),
    "Intel(R) Xeon(R) Platinum 8580": (350.0, 120),
    "Intel(R) Xeon(R) Platinum 8480+": (350.0, 112),
    "Intel(R) Xeon(R) Platinum 8480C": (350.0, 112),
    "Intel(R) Xeon(R) Platinum 8468": (350.0, 96),
    "Intel(R) Xeon(R) Platinum 8462Y+": (300.0, 64),
    "Intel(R) Xeon(R) 6960P": (500.0, 144),
    "Intel(R) Xeon(R) 6767P": (350.0, 128),
    "AMD EPYC 9654 96-Core Processor": (360.0, 192),
    "AMD EPYC 9554 64-Core Processor": (360.0, 128),
    "AMD EPYC 9534 64-Core Processor": (280.0, 128),
    "AMD EPYC 9454 48-Core Processor": (290.0, 96),
    "AMD EPYC 9474F 48-Core Processor": (360.0, 96),
    "AMD EPYC 9575F 64-Core Processor": (400.0, 128),
    "AMD EPYC 9655 96-Core Processor": (400.0, 192),
    "AMD EPYC 9755 128-Core Processor": (500.0, 256),
}


# Virtualised hosts often report a generic model name ("Intel(R) Xeon(R)
# Processor"): fall back to the CPU generation (vendor, family, model) and
# the flagship B200-host part of that generation.
CPU_GEN_TDP = {
    ("GenuineIntel", 6, 143): (350.0, 112, "Sapphire Rapids; Xeon Platinum 8480+-class"),
    ("GenuineIntel", 6, 207): (350.0, 120, "Emerald Rapids; Xeon Platinum 8570/8580-class"),
    ("GenuineIntel", 6, 173): (500.0, 256, "Granite Rapids; Xeon 6980P-class"),
    ("AuthenticAMD", 25, 17): (360.0, 192, "Genoa; EPYC 9654-class"),
    ("AuthenticAMD", 26, 2): (500.0, 256, "Turin; EPYC 9755-class"),
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--mode", choices=["fast", "exact"], default="fast")
    ap.add_argument("--config", choices=sorted(CONFIGS), default="config2")
    ap.add_argument("--kernels", type=int, default=None, help="override the kernel count (config5 sweep)")
    ap.add_argument("--series", type=int, default=None, help="override series per GPU (total for config3)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-public", action="store_true", help="skip the numpy transform() e2e legs")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-variants", action="store_true", help="skip the MPV / float64 throughput lines")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    return ap.parse_args()


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


def host_cpu():
    """Model name, usable threads and the nominal power share they stand for."""
    fields = {}
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if not ln.strip():
                    break  # first processor only
                k, _, v = ln.partition(":")
                fields[k.strip()] = v.strip()
    except OSError:
        pass
    model = fields.get("model name")
    threads = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)
    tdp = CPU_TDP.get(model or "")
    info = {"model": model, "vendor": fields.get("vendor_id"), "family": fields.get("cpu family"),
            "model_number": fields.get("model"), "threads_usable": threads, "threads_online": os.cpu_count()}
    source = "model name"
    if not tdp:
        try:
            gen = CPU_GEN_TDP.get((fields.get("vendor_id"), int(fields.get("cpu family", -1)),
                                   int(fields.get("model", -1))))
        except ValueError:
            gen = None
        if gen:
            tdp = gen[:2]
            source = f"CPU generation ({gen[2]})"
    if tdp:
        pkg_w, pkg_threads = tdp
        info.update({"package_tdp_w": pkg_w, "package_threads": pkg_threads, "tdp_source": source,
                     "nominal_w_used": pkg_w * min(1.0, threads / pkg_threads),
                     "nominal_w_note": "package TDP x (threads used / threads per package), nominal (no RAPL)"})
    else:
        info.update({"nominal_w_used": None, "nominal_w_note": "CPU model not in bench.CPU_TDP"})
    return info


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

    threads = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)
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
    """--impl reference: the reference algorithm on the host cores.  Only
    oracle/ is loaded (the bank is drawn through numpy, as the reference
    does, so the product library never enters this process)."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    import oracle.oracle as orc
    from paper_2601_17091_b200 import GenOptions, generate_bank, synth_random

    orc.build()
    bank = generate_bank(cfg["l"], cfg["c"], cfg["k"], GenOptions(seed=0), native=False)
    threads = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)
    if args.config == "config1":
        # configs[0]: the whole CPU pipeline (transform + ridge) per step
        runs = [cpu_config1(bank, cfg) for _ in range(max(1, args.steps))]
        total = sum(r["seconds"] for r in runs)
        value = cfg["n"] * len(runs) / total
        line = {"impl": "reference", "metric": "ROCKET transform + ridge fit series/sec (FordA shape, 10k kernels)",
                "value": value, "unit": "series/s", "n_gpus": world, "steps": len(runs), "warmup": 0,
                "ms_per_step": 1e3 * total / len(runs), "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "f32 transform, f64 ridge",
                "data": "synthetic: synth_two_class(1801, 500, seed=1)[:3601] with its labels",
                "config": {"workload": cfg["workload"], "series": cfg["n"], "parallelism": "cpu threads"},
                "cpu_baseline": {"value": value, "unit": "series/s", "cores": threads, "kind": "port",
                                 "sample": "the whole pipeline per step", "host_cpu": host_cpu()},
                "e2e": {"value": value, "unit": "series/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return
    # one step = a bounded sample sized for ~2.5 s of CPU work
    rate, _, _, _ = cpu_sample_rate(bank, cfg, 2.5)
    m = max(threads, int(rate * 2.5 // threads) * threads)
    x = synth_random(m, cfg["c"], cfg["l"], seed=1).values
    for _ in range(args.warmup):
        orc.oracle_transform(x[:threads], bank, nthreads=threads)
    times = []
    from paper_2601_17091_b200.engine import expected_dot_products

    for _ in range(args.steps):
        t0 = time.perf_counter()
        _, executed = orc.oracle_transform(x, bank, nthreads=threads, return_executed=True)
        times.append(time.perf_counter() - t0)
        assert executed == expected_dot_products(bank, m)
    total = sum(times)
    value = m * args.steps / total
    cpu = host_cpu()
    fpk = 2
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "series/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps,
        "higher_is_better": True, "scaling": cfg["scaling"], "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (synth_random seed 1; bank generate_bank seed 0 via numpy)",
        "config": {"workload": cfg["workload"], "series_per_step": m, "l_series": cfg["l"],
                   "n_channels": cfg["c"], "n_kernels": cfg["k"], "parallelism": "cpu threads"},
        "cpu_baseline": {"value": value, "unit": "series/s", "cores": threads, "kind": "port",
                         "sample": f"{m} series per step of the {cfg['workload']} workload",
                         "host_cpu": cpu},
        "energy": {"nominal_w": cpu["nominal_w_used"],
                   "features_per_joule_nominal": (value * bank.count * fpk / cpu["nominal_w_used"])
                   if cpu["nominal_w_used"] else None},
        "e2e": {"value": value, "unit": "series/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def config1_data(cfg):
    """BASELINE configs[0]: synth_two_class(1801, 500, seed=1)[:3601] (SURVEY
    §8d), labels included."""
    from paper_2601_17091_b200 import synth_two_class

    ds = synth_two_class((cfg["n"] + 1) // 2, cfg["l"], seed=1)
    return ds.values[: cfg["n"]], ds.labels[: cfg["n"]]


def cpu_config1(bank, cfg):
    """The whole config-1 pipeline on the host cores: the C port of the
    transform (all threads) + the numpy/LAPACK restatement of the
    reference's ridge.fit and predict (oracle/ridge_oracle.py)."""
    import oracle.oracle as orc
    from oracle import ridge_oracle

    values, labels = config1_data(cfg)
    threads = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)
    orc.oracle_transform(values[:threads], bank, nthreads=threads)  # warm
    t0 = time.perf_counter()
    feats = orc.oracle_transform(values, bank, nthreads=threads)
    t1 = time.perf_counter()
    model = ridge_oracle.fit(feats, labels, alpha=1.0)
    pred = ridge_oracle.predict(model, feats)
    t2 = time.perf_counter()
    acc = float(np.mean(pred == np.asarray(labels)))
    return {"seconds": t2 - t0, "transform_s": t1 - t0, "ridge_s": t2 - t1, "threads": threads,
            "train_accuracy": acc, "value": len(labels) / (t2 - t0)}


def run_config1(args, cfg):
    """configs[0] on the GPU: transform (features stay in HBM) + ridge fit +
    predict per step; the CPU leg runs the same pipeline on the host."""
    import torch

    from paper_2601_17091_b200 import GenOptions, device_bank, generate_bank, ridge

    torch.cuda.set_device(0)
    values, labels = config1_data(cfg)
    n = len(labels)
    bank = generate_bank(cfg["l"], cfg["c"], cfg["k"], GenOptions(seed=0))
    db = device_bank(bank, 0)
    info = db.info
    x_host = torch.from_numpy(values).pin_memory()
    x_dev = x_host.cuda()
    feats = torch.empty((n, 2 * bank.count), device="cuda")
    stream = torch.cuda.current_stream()
    expected = None
    from paper_2601_17091_b200.engine import expected_dot_products

    expected = expected_dot_products(bank, n)
    stages = {}

    def step(xd, timed_stages=False):
        e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        e[0].record(stream)
        ex = db.transform_into(xd.data_ptr(), n, feats.data_ptr(), feats.shape[1], mode=args.mode,
                               stream=stream.cuda_stream)
        e[1].record(stream)
        model = ridge.fit(feats, labels, alpha=1.0)
        e[2].record(stream)
        pred = ridge.predict(model, feats)  # labels on the host
        e[3].record(stream)
        if timed_stages:
            torch.cuda.synchronize()
            stages.update(transform_ms=e[0].elapsed_time(e[1]), ridge_fit_ms=e[1].elapsed_time(e[2]),
                          predict_ms=e[2].elapsed_time(e[3]))
        if ex != expected:
            raise RuntimeError("executed positions differ from expected_dot_products")
        return pred

    for _ in range(args.warmup):
        step(x_dev)
    pred = step(x_dev, timed_stages=True)
    acc = float(np.mean(pred == np.asarray(labels)))
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(0) as clk:
        e0.record(stream)
        for _ in range(args.steps):
            step(x_dev)
        e1.record(stream)
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    value = n * args.steps / (ms / 1e3)
    # e2e: the series from pinned host memory each step, predictions read back
    t0 = time.perf_counter()
    for _ in range(args.steps):
        xd = x_host.to("cuda", non_blocking=True)
        step(xd)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    cpu = None
    if not args.no_cpu:
        import oracle.oracle as orc

        orc.build()
        c = cpu_config1(bank, cfg)
        cpu = {"value": c["value"], "unit": "series/s", "cores": c["threads"], "kind": "port",
               "sample": f"the whole config-1 pipeline ({n} series): transform {c['transform_s']:.1f} s (C port of "
                         f"engine._run_batch) + ridge fit/predict {c['ridge_s']:.2f} s (numpy/LAPACK restatement "
                         f"of ridge.py:100-197)", "train_accuracy": c["train_accuracy"], "host_cpu": host_cpu()}
    flops = info["useful_flops_per_series"] * n / (stages["transform_ms"] / 1e3) / 1e12
    line = {
        "metric": "ROCKET transform + ridge fit series/sec (FordA shape, 10k kernels)", "value": value,
        "unit": "series/s", "n_gpus": 1, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32 transform, f64 ridge",
        "mode": args.mode, "data": "synthetic: synth_two_class(1801, 500, seed=1)[:3601] with its labels",
        "config": {"workload": cfg["workload"], "series": n, "l_series": cfg["l"], "n_kernels": bank.count,
                   "ridge": "fp64 one-vs-rest, dual Cholesky on the GPU (features never leave HBM)"},
        "stages": stages, "train_accuracy": acc,
        "roofline": {"bound": "fp32", "achieved": flops, "peak": FP32_PEAK_MEASURED, "unit": "TFLOP/s",
                     "frac": flops / FP32_PEAK_MEASURED, "traffic": None,
                     "kernel": "rocket_wide_kernel (the transform stage; the ridge stage is cuBLAS/cuSOLVER fp64)"},
        "e2e": {"value": n * args.steps / dt, "unit": "series/s", "h2d_bytes_per_step": int(x_host.numel() * 4),
                "d2h_bytes_per_step": int(n * 8), "ms_per_step": 1e3 * dt / args.steps},
        "cpu_baseline": cpu, "clocks": clk.summary(), "gpu_launches": int(info["n_launches"]) * args.steps,
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
    if args.config == "config1":
        return run_config1(args, cfg)

    import torch
    import torch.distributed as dist

    from paper_2601_17091_b200 import GenOptions, device_bank, generate_bank, synth_random, transform
    from paper_2601_17091_b200.engine import expected_dot_products, plan_shards

    rank, world, local = dist_env()
    # one process per GPU; the modulo only matters for a logic check of the
    # multi-rank path on a box with fewer GPUs than ranks (gloo backend)
    local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    backend = os.environ.get("RK_BENCH_BACKEND", "nccl")
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)

    def reduce(value, op):
        """All-reduce a host float over ranks (device tensor for NCCL)."""
        if world == 1:
            return value
        t = torch.tensor([value], dtype=torch.float64, device="cuda" if backend == "nccl" else "cpu")
        dist.all_reduce(t, op={"max": dist.ReduceOp.MAX, "sum": dist.ReduceOp.SUM}[op])
        return float(t.item())

    def barrier():
        if world > 1:
            dist.barrier()

    bank = generate_bank(cfg["l"], cfg["c"], cfg["k"], GenOptions(seed=0))
    db = device_bank(bank, local)
    info = db.info
    fpk = 2
    if cfg["scaling"] == "strong":
        # configs[2]: the whole job's series split by plan_shards; each rank
        # synthesises its own shard (seed 1 + shard)
        total_n = cfg["n"]
        row0, n = plan_shards(total_n, world)[rank]
    else:
        row0, n = 0, cfg["n"]
        total_n = n * world
    values = synth_random(n, cfg["c"], cfg["l"], seed=1 + rank).values  # pageable numpy, as a user holds it
    x_host = torch.from_numpy(values).pin_memory()
    x_dev = x_host.cuda()
    out_dev = torch.empty((n, bank.count * fpk), device="cuda", dtype=torch.float32)
    stream = torch.cuda.Stream()
    sptr = stream.cuda_stream
    expected = expected_dot_products(bank, n)

    def step(mode, xp, op):
        return db.transform_into(xp, n, op, bank.count * fpk, mode=mode, stream=sptr)

    def timed(mode):
        """W warm-up + K timed device-resident transforms.  Returns the max
        over ranks of the CUDA-event time and the NVML energy of the timed
        steps summed over ranks (None without NVML)."""
        for _ in range(args.warmup):
            step(mode, x_dev.data_ptr(), out_dev.data_ptr())
        torch.cuda.synchronize()
        barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        mj0 = nvml_energy_mj(local)
        e0.record(stream)
        executed = []
        for _ in range(args.steps):
            executed.append(step(mode, x_dev.data_ptr(), out_dev.data_ptr()))
        e1.record(stream)
        torch.cuda.synchronize()
        mj1 = nvml_energy_mj(local)
        barrier()
        bad = [e for e in executed if e != expected]
        if bad:
            raise RuntimeError(f"executed positions {bad[0]} != expected_dot_products {expected}")
        ms = reduce(e0.elapsed_time(e1), "max")
        joules = reduce((mj1 - mj0) / 1e3, "sum") if mj0 is not None and mj1 is not None else None
        return ms, joules

    # ---- headline: device-resident, selected mode -------------------------
    with ClockSampler(local) as clk:
        ms_total, joules = timed(args.mode)
    ms_step = ms_total / args.steps
    total_series = total_n * args.steps
    value = total_series / (ms_total / 1e3)
    flops_series = info["useful_flops_per_series"]
    achieved_tflops = flops_series * n / (ms_step / 1e3) / 1e12

    # ---- the other mode, same protocol -----------------------------------
    other = "exact" if args.mode == "fast" else "fast"
    ms_other, joules_other = timed(other)

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
            ex = db.transform_into(xv.data_ptr(), nv, ov.data_ptr(), bank.count * fpk_v, mode=mode_v, fpk=fpk_v,
                                   precision=prec, stream=sptr)
            ev1.record(stream)
            torch.cuda.synchronize()
            assert ex == expected_dot_products(bank, nv)
            variants[name] = {"value": nv / (ev0.elapsed_time(ev1) / 1e3), "unit": "series/s", "series": nv,
                              "fpk": fpk_v, "precision": prec, "mode": mode_v}
            del xv, ov

    # ---- e2e through the public C-ABI call with pinned host buffers --------
    e2e = None
    if not args.no_e2e:
        del out_dev
        torch.cuda.empty_cache()
        blk = min(n, E2E_BLOCK) if cfg["scaling"] == "strong" else n
        out_host = torch.empty((blk, bank.count * fpk), dtype=torch.float32).pin_memory()

        def e2e_step():
            ex = 0
            for s0 in range(0, n, blk):
                cnt = min(blk, n - s0)
                ex += db.transform_into(x_host.data_ptr() + s0 * cfg["c"] * cfg["l"] * 4, cnt,
                                        out_host.data_ptr(), bank.count * fpk, mode=args.mode)
                _ = float(out_host[cnt - 1, 1])  # the block's result read on the host
            return ex

        e2e_step()
        barrier()
        with ClockSampler(local) as clk_e2e:
            t0 = time.perf_counter()
            for _ in range(args.steps):
                if e2e_step() != expected:
                    raise RuntimeError("e2e executed positions differ from expected_dot_products")
            dt = time.perf_counter() - t0
        dt = reduce(dt, "max")
        e2e = {"value": total_series / dt, "unit": "series/s",
               "h2d_bytes_per_step": int(x_host.numel() * 4),
               "d2h_bytes_per_step": int(n * bank.count * fpk * 4),
               "ms_per_step": 1e3 * dt / args.steps,
               "clocks": clk_e2e.summary(),
               "path": "DeviceBank.transform_into -> rk_transform (host pinned x/out, pipelined H2D/kernel/D2H)"
                       + (f", {blk}-row calls into one reused pinned output block" if blk < n else "")}
        del out_host

    # ---- e2e through the reference-facing numpy transform() ----------------
    e2e_public = None
    if not args.no_public and cfg["scaling"] == "weak":
        e2e_public = {"path": "paper_2601_17091_b200.transform(numpy pageable (n, C, L)) -> FeatureMatrix "
                              "(the reference's engine.transform surface, engine.py:324-333)",
                      "steps": min(args.steps, 3)}
        for mode in ("fast", "exact"):
            transform(values, bank, mode=mode)  # untimed: sizes the pinned ring and its copy threads
            barrier()
            t0 = time.perf_counter()
            for _ in range(e2e_public["steps"]):
                fm = transform(values, bank, mode=mode)
                _ = float(fm.values[n - 1, 1])
                del fm
            dt = reduce(time.perf_counter() - t0, "max")
            e2e_public[mode] = n * world * e2e_public["steps"] / dt
        e2e_public["unit"] = "series/s"

    # ---- CPU baseline on rank 0 at N=1 -------------------------------------
    cpu = None
    cpu_info = host_cpu()
    if rank == 0 and world == 1 and not args.no_cpu:
        import oracle.oracle as orc

        orc.build()
        rate, m, dt, threads = cpu_sample_rate(bank, cfg, args.cpu_seconds)
        cpu = {"value": rate, "unit": "series/s", "cores": threads, "kind": "port",
               "sample": f"{m} series of the same workload (synth_random seed 1), {dt:.1f} s, "
                         "oracle/rocket_oracle.c restating engine._run_batch, pthreads",
               "host_cpu": cpu_info}

    # ---- energy: measured GPU features/J, the paper's nominal per-watt gain
    energy = None
    feats = total_series * bank.count * fpk
    if joules:
        energy = {"joules_all_ranks": joules, "window": "NVML total-energy counter read right before the first "
                                                        "and right after the last timed step, summed over ranks",
                  "features_per_joule": feats / joules,
                  "gpu_avg_w_per_gpu": joules / (ms_total / 1e3) / world}
        if joules_other:
            energy["features_per_joule_" + other] = feats / joules_other
    if cpu is not None and energy is not None and cpu_info["nominal_w_used"]:
        cpu_w = cpu_info["nominal_w_used"]
        cpu_fpj = cpu["value"] * bank.count * fpk / cpu_w
        speedup = value / cpu["value"]
        energy.update({
            "cpu_nominal_w": cpu_w,
            "cpu_features_per_joule_nominal": cpu_fpj,
            "gpu_nominal_w": GPU_NOMINAL_W * world,
            "speedup_vs_cpu": speedup,
            # the paper's metric: speedup x nominal watts ratio (bench.per_watt_gain)
            "per_watt_gain": speedup * cpu_w / (GPU_NOMINAL_W * world),
            "per_watt_gain_measured_gpu": (feats / joules) / cpu_fpj,
            "per_watt_note": "per_watt_gain = speedup x CPU nominal W / GPU nominal W (reference bench.py:62-70, "
                             "PAPER.md:106); _measured_gpu uses NVML joules for the GPU, nominal for the CPU",
        })

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
            "scaling": cfg["scaling"],
            "vs_baseline": None,
            "dtype": "f32",
            "mode": args.mode,
            "data": "synthetic: synth_random(seed=1+rank) float32 series, generate_bank(seed=0) kernels",
            "config": {"workload": cfg["workload"], "series_total": total_n, "series_per_gpu": n,
                       "l_series": cfg["l"], "n_channels": cfg["c"], "n_kernels": bank.count,
                       "parallelism": f"series-sharded x{world}",
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
            "e2e_public": e2e_public,
            "variants": variants,
            "cpu_baseline": cpu,
            "clocks": clk.summary(),
            "energy": energy,
            "executed_checked": f"every timed step: executed == expected_dot_products = {expected}",
            "gpu_launches": int(info["n_launches"]) * args.steps,
            "bank": {"groups": info["n_groups"], "chunks": info["n_chunks"], "half_warp_chunks": info["n_half_chunks"],
                     "launches_per_step": info["n_launches"], "smem_bytes": info["smem_bytes"],
                     "path": {0: "class", 1: "wide", 2: "wide (series in global memory)"}[info["path"]],
                     "ctas_per_sm": info["ctas_per_sm"]},
        }
        if world > 1:
            line["backend"] = backend
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
