#!/bin/bash
# e2e (pinned host buffers) of the FordA shape against the row-batch split of
# rk_transform's pinned pipeline: RK_E2E_MIN_ROWS / RK_E2E_BATCHES.
mkdir -p gpurun_out/e2e_sweep
for cfg in "4096 6" "1000 2" "1000 3" "1000 4" "1000 6"; do
  set -- $cfg
  RK_E2E_MIN_ROWS=$1 RK_E2E_BATCHES=$2 python bench.py --config forda --no-cpu --no-variants \
    > gpurun_out/e2e_sweep/forda_$1_$2.json 2> gpurun_out/e2e_sweep/forda_$1_$2.err
  python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[1], round(d['value']), round(d['e2e']['value']))" gpurun_out/e2e_sweep/forda_$1_$2.json
done
