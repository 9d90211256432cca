"""profiles/ncu_summary_<config>.json from an ncu launch list with DRAM bytes
of tools/profile_transform.py (two transforms; the second is measured).

    python tools/dram_summary.py <launches.csv> <config> <series> <out.json>
"""
import csv
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

src, cfg_name, series, dst = sys.argv[1], sys.argv[2], int(sys.argv[3]), sys.argv[4]
rows = list(csv.reader(open(src)))
hdr, recs, order = None, {}, []
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if "rocket" not in d["Kernel Name"]:
            continue
        if d["ID"] not in recs:
            recs[d["ID"]] = {}
            order.append(d["ID"])
        recs[d["ID"]][d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
ks = [recs[k] for k in order]
ks = ks[len(ks) // 2:]  # the measured (second) transform
rd = sum(k.get("dram__bytes_read.sum", 0) for k in ks)
wr = sum(k.get("dram__bytes_write.sum", 0) for k in ks)
t = sum(k.get("gpu__time_duration.sum", 0) for k in ks)
from bench import CONFIGS  # noqa: E402

c = CONFIGS[cfg_name]
alg = 4 * c["c"] * c["l"] + 8 * c["k"]
out = {
    "config": f"{cfg_name} bank ({c['k']} kernels, C={c['c']}, L={c['l']}), {series} series, fast mode, "
              f"one transform = {len(ks)} launches",
    "command": "ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none "
               f"--csv python tools/profile_transform.py --config {cfg_name} --series {series} (second transform)",
    "launches": len(ks),
    "dram_read_bytes": rd, "dram_write_bytes": wr,
    "dram_bytes_per_series": (rd + wr) / series,
    "dram_read_per_series": rd / series, "dram_write_per_series": wr / series,
    "algorithmic_bytes_per_series": alg,
    "traffic_over_algorithmic": (rd + wr) / series / alg,
    "serialised_ns": t,
}
json.dump(out, open(dst, "w"), indent=1)
print(json.dumps(out, indent=1))
