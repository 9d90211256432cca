set -x
mkdir -p gpurun_out/ab
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for c in config2 forda config4 uni2048 config5; do
  for v in half nohalf; do
    if [ $v = nohalf ]; then export RK_NO_HALF=1; else unset RK_NO_HALF; fi
    timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-e2e --no-cpu --no-variants > gpurun_out/ab/${c}_$v.json 2> gpurun_out/ab/${c}_$v.err
    python -c "import json;d=json.load(open('gpurun_out/ab/${c}_$v.json'));print('$c','$v',d['value'],d.get('bank',{}).get('launches_per_step'))"
  done
done
