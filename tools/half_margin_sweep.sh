#!/bin/bash
# Sweep the half-warp chunk margin of the cost model (RK_HALF_MARGIN, percent:
# a chunk runs half-warp when its modelled cost is below margin% of the best
# full-warp option), device-resident fast mode.
mkdir -p gpurun_out/hm
for c in config2 forda uni2048; do
  for m in 90 101 110 120 135; do
    RK_HALF_MARGIN=$m timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-e2e --no-cpu --no-variants \
      > gpurun_out/hm/${c}_$m.json 2> gpurun_out/hm/${c}_$m.err
    python -c "import json;d=json.load(open('gpurun_out/hm/${c}_$m.json'));print('$c', $m, round(d['value']), round(d['other_mode']['value']))"
  done
done
