"""Condense ncu outputs into profiles/ summaries.

    python tools/ncu_summary.py launches <launches.csv> <out.json>
    python tools/ncu_summary.py report <prof.ncu-rep> <out.txt>
    python tools/ncu_summary.py bench <launches.csv> <out.json>   (a whole bench.py run, per kernel name)
"""
import csv
import json
import re
import subprocess
import sys


def launches(src, dst, skip_first_half=True):
    rows = list(csv.reader(open(src)))
    hdr = None
    recs = {}
    order = []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            key = d["ID"]
            if key not in recs:
                recs[key] = {"kernel": d["Kernel Name"]}
                order.append(key)
            try:
                recs[key][d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
            except ValueError:
                recs[key][d["Metric Name"]] = d["Metric Value"]
    ks = [recs[k] for k in order if "rocket" in recs[k]["kernel"]]
    if skip_first_half:  # profile_transform.py runs one warm-up transform first
        ks = ks[len(ks) // 2:]
    tot = sum(k.get("gpu__time_duration.sum", 0) for k in ks)
    out = {"launches": len(ks), "total_ns": tot, "kernels": []}
    for k in ks:
        t = k.get("gpu__time_duration.sum", 0)
        out["kernels"].append({
            "kernel": re.sub(r"\(rk::\w+\)|void |rk::", "", k["kernel"]),
            "ns": t, "share": t / tot if tot else 0,
            "fma_pipe_pct": k.get("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"),
            "issue_pct": k.get("smsp__issue_active.avg.pct_of_peak_sustained_active"),
            "dram_bytes": (k.get("dram__bytes_read.sum", 0) or 0) + (k.get("dram__bytes_write.sum", 0) or 0),
        })
    json.dump(out, open(dst, "w"), indent=1)
    print(f"{len(ks)} launches, {tot/1e6:.2f} ms total")


WANT = [
    "gpu__time_duration.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "launch__block_size",
    "launch__grid_size", "launch__occupancy_limit_shared_mem", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "smsp__inst_executed.sum",
    "smsp__thread_inst_executed_per_inst_executed.ratio",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum", "smsp__sass_inst_executed_op_shared_ld.sum",
    "derived__memory_l1_conflicts_shared_nway", "derived__memory_l1_wavefronts_shared_excessive",
    "smsp__sass_branch_targets_threads_divergent.sum", "smsp__sass_branch_targets.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
]


def report(src, dst):
    raw = subprocess.run(["ncu", "-i", src, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    hdr = rows[0]
    lines = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        lines.append(f"kernel: {d['Kernel Name']}")
        for w in WANT:
            if w in d:
                lines.append(f"  {w} = {d[w]}")
        st = []
        for k in hdr:
            if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued"):
                try:
                    st.append((float(d[k].replace(",", "")), k.replace("smsp__pcsamp_warps_issue_stalled_", "")))
                except ValueError:
                    pass
        st.sort(reverse=True)
        tot = sum(v for v, _ in st) or 1
        lines.append("  stall samples (share): " + ", ".join(f"{k} {v/tot:.1%}" for v, k in st[:8]))
    src_csv = subprocess.run(["ncu", "-i", src, "--page", "source", "--csv", "--print-source", "sass"],
                             capture_output=True, text=True).stdout
    srows = list(csv.reader(src_csv.splitlines()[1:]))
    if srows:
        sh = srows[0]
        ops = {}
        for r in srows[1:]:
            if len(r) != len(sh):
                continue
            d = dict(zip(sh, r))
            m = re.match(r"\s*(@!?U?P\w+\s+)?([A-Z0-9_]+)", d["Source"])
            if m:
                try:
                    ops[m.group(2)] = ops.get(m.group(2), 0) + float(d["Instructions Executed"] or 0)
                except ValueError:
                    pass
        f = ops.get("FFMA2", 1) or 1
        lines.append("  executed instructions per FFMA2: " + ", ".join(
            f"{k} {v / f:.3f}" for k, v in sorted(ops.items(), key=lambda kv: -kv[1])[:16]))
    open(dst, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


def bench(src, dst):
    """Launch list of a whole `bench.py` run under ncu: per-kernel-name launch
    counts, total and mean durations, and each name's share of the
    library's GPU time (the serialised, cold-cache ncu times)."""
    launches(src, dst + ".tmp", skip_first_half=False)
    data = json.load(open(dst + ".tmp"))
    import os

    os.remove(dst + ".tmp")
    agg = {}
    for k in data["kernels"]:
        name = k["kernel"].split("(")[0]
        a = agg.setdefault(name, {"kernel": name, "launches": 0, "ns": 0.0})
        a["launches"] += 1
        a["ns"] += k["ns"]
    tot = sum(a["ns"] for a in agg.values()) or 1
    rows = sorted(agg.values(), key=lambda a: -a["ns"])
    for a in rows:
        a["share"] = a["ns"] / tot
        a["mean_ns"] = a["ns"] / a["launches"]
    json.dump({"launches": data["launches"], "total_ns": tot, "by_kernel": rows, "per_launch": data["kernels"]},
              open(dst, "w"), indent=1)
    for a in rows:
        print(f"{a['kernel'][:70]:70s} {a['launches']:5d} {a['ns']/1e6:9.2f} ms {a['share']:.1%}")


if __name__ == "__main__":
    {"launches": launches, "report": report, "bench": bench}[sys.argv[1]](sys.argv[2], sys.argv[3])
