#!/bin/bash
# A/B of one environment switch on the device-resident bench lines.
#   tools/ab_env.sh <VAR=value> <tag> [config[:kernels] ...]
# prints value (series/s) and TFLOP/s per config with and without the switch.
set -u
var=$1; tag=$2; shift 2
mkdir -p gpurun_out/ab
for c in "$@"; do
  cfg=${c%%:*}; k=""
  [[ "$c" == *:* ]] && k="--kernels ${c##*:}"
  for side in base test; do
    if [ $side = test ]; then envs="$var"; else envs=""; fi
    env $envs python bench.py --config $cfg $k --steps 5 --warmup 3 --no-e2e --no-public --no-cpu --no-variants \
      > gpurun_out/ab/${tag}_${cfg}${k:+_k${c##*:}}_$side.json 2> gpurun_out/ab/${tag}_${cfg}_$side.err
    python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[2], sys.argv[3], round(d['value']), round(d['roofline']['achieved'],2), round(d['roofline']['frac'],3), 'exact', round(d['other_mode']['value']))" gpurun_out/ab/${tag}_${cfg}${k:+_k${c##*:}}_$side.json "$c" $side
  done
done
