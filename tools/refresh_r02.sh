#!/bin/bash
# Round-2 measurement set (GPU box, repo root): the driver's bench command,
# every config's bench line, the reference arm, the config-5 kernel sweep.
set -u
mkdir -p gpurun_out/r02
python bench.py --steps 20 --warmup 5 > gpurun_out/r02/bench_config2.json 2> gpurun_out/r02/bench_config2.err
python bench.py --impl reference --steps 5 --warmup 2 > gpurun_out/r02/bench_reference.json 2> gpurun_out/r02/bench_reference.err
for c in config4 config5 uni2048 forda; do
  python bench.py --config $c --steps 10 --warmup 3 --no-public > gpurun_out/r02/bench_$c.json 2> gpurun_out/r02/bench_$c.err
done
python bench.py --config config3 --steps 3 --warmup 3 --no-variants > gpurun_out/r02/bench_config3.json 2> gpurun_out/r02/bench_config3.err
for k in 1000 2000 5000 20000 50000 100000; do
  python bench.py --config config5 --kernels $k --steps 3 --warmup 3 --no-e2e --no-public --no-cpu --no-variants \
    > gpurun_out/r02/bench_config5_k$k.json 2> gpurun_out/r02/bench_config5_k$k.err
done
echo done
