#!/bin/bash
# Sweep the R-choice cost model knobs on config 2 (device-resident, fast).
for m in 100 70 130 160; do
  RK_MASK_COST_PCT=$m python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print('mask_pct=$m', round(d['value']), round(d['other_mode']['value']))"
done
