#!/bin/bash
# config 2 e2e (pinned host buffers) against the pinned pipeline's batch count.
mkdir -p gpurun_out/e2e_sweep2
for nb in 6 10 16 24; do
  RK_E2E_BATCHES=$nb python bench.py --config config2 --no-cpu --no-variants --steps 5 \
    > gpurun_out/e2e_sweep2/config2_$nb.json 2> gpurun_out/e2e_sweep2/config2_$nb.err
  python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[1], round(d['value']), round(d['e2e']['value']), round(d['e2e']['ms_per_step'],2))" gpurun_out/e2e_sweep2/config2_$nb.json
done
