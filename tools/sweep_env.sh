#!/bin/bash
# Device-resident bench lines for a list of environment settings.
#   tools/sweep_env.sh <config> "<ENV=.. ENV=..>" ["<ENV=..>" ...]
set -u
cfg=$1; shift
mkdir -p gpurun_out/sweep
i=0
for envs in "$@"; do
  i=$((i + 1))
  env $envs python bench.py --config $cfg --steps 5 --warmup 3 --no-e2e --no-public --no-cpu --no-variants \
    > gpurun_out/sweep/${cfg}_$i.json 2> gpurun_out/sweep/${cfg}_$i.err
  python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[2], '|', sys.argv[3], round(d['value']), round(d['roofline']['frac'],3), 'exact', round(d['other_mode']['value']))" gpurun_out/sweep/${cfg}_$i.json $cfg "$envs"
done
