#!/bin/bash
# Round-2 profile set (GPU box, repo root; ncu only after the plain runs exit 0).
set -u
mkdir -p gpurun_out/prof2
B="python bench.py --steps 2 --warmup 3 --no-variants --no-public --no-cpu"
$B > gpurun_out/prof2/bench_plain.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/prof2/launches_bench.csv \
  $B > gpurun_out/prof2/ncu_bench.log 2>&1
for c in config2:20000 forda:3601 config5:10000 config4:4000 uni2048:10000; do
  cfg=${c%%:*}; n=${c##*:}
  python tools/profile_transform.py --config $cfg --series $n > gpurun_out/prof2/plain_$cfg.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/prof2/dram_$cfg.csv python tools/profile_transform.py --config $cfg --series $n \
    > gpurun_out/prof2/ncu_dram_$cfg.log 2>&1
done
tools/ncu_top_launch.sh config2_r02 --config config2 --series 20000
echo refresh done
