#!/bin/bash
# Round-end measurement set (run on the GPU box from the repo root):
# bench lines for every config + the reference arm, the ncu launch list of
# a whole bench run, one ncu --set full capture of the largest fast-mode
# class launch, and per-transform DRAM bytes.
set -u
mkdir -p gpurun_out/refresh
for c in config2 config4 config5 uni2048 forda; do
  python bench.py --config $c > gpurun_out/refresh/bench_$c.json 2> gpurun_out/refresh/bench_$c.err || tail -3 gpurun_out/refresh/bench_$c.err
done
python bench.py --impl reference > gpurun_out/refresh/bench_reference.json 2> gpurun_out/refresh/bench_reference.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/refresh/launches_bench.csv \
  python bench.py --steps 2 --warmup 3 --no-variants > gpurun_out/refresh/ncu_bench.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/refresh/launches_dram.csv python tools/profile_transform.py --series 20000 > /dev/null 2>&1
# the largest fast-mode class launch of the measured (second) transform
python - <<'PY' > gpurun_out/refresh/skip.txt
import csv
rows = [r for r in csv.reader(open("gpurun_out/refresh/launches_dram.csv")) if len(r) > 5]
h = rows[0]
ks = {}
for r in rows[1:]:
    d = dict(zip(h, r))
    if "rocket" in d["Kernel Name"] and d["Metric Name"] == "gpu__time_duration.sum":
        ks[int(d["ID"])] = float(d["Metric Value"])
ids = sorted(ks)
half = ids[len(ids) // 2:]
best = max(half, key=lambda i: ks[i])
print(ids.index(best))
PY
SKIP=$(cat gpurun_out/refresh/skip.txt)
ncu --set full --clock-control none --import-source on -k regex:rocket_wide_kernel -s $SKIP -c 1 \
  -o gpurun_out/refresh/wide_full python tools/profile_transform.py --series 20000 > gpurun_out/refresh/ncu_full.log 2>&1
echo "refresh done, full capture at launch index $SKIP"
