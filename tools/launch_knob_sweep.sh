#!/bin/bash
# Wide-launch knobs after half-warp chunks: series per item (RK_SPI, max),
# CTAs per SM (RK_WIDE_CTAS), min items per CTA slot (RK_MIN_ITEMS);
# device-resident, both modes.
mkdir -p gpurun_out/knobs
run() {  # name env...
  local name=$1; shift
  for c in config2 forda; do
    env "$@" timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-e2e --no-cpu --no-variants \
      > gpurun_out/knobs/${c}_$name.json 2> gpurun_out/knobs/${c}_$name.err
    python -c "import json;d=json.load(open('gpurun_out/knobs/${c}_$name.json'));print('$c', '$name', round(d['value']), round(d['other_mode']['value']))"
  done
}
run default RK_NONE=1
run spi4 RK_SPI=4
run spi12 RK_SPI=12
run spi16 RK_SPI=16
run ctas5 RK_WIDE_CTAS=5
run ctas7 RK_WIDE_CTAS=7
run items1 RK_MIN_ITEMS=1
run items3 RK_MIN_ITEMS=3
