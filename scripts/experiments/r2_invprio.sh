#!/bin/bash
export PYTHONPATH=. SPD_WATCHDOG=900
for v in -1 0 -1 0 -2 0; do
  SPDKFAC_INV_PRIORITY=$v timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/r2ip.json 2>gpurun_out/r2ip.err
  python -c "import json;d=json.loads(open('gpurun_out/r2ip.json').read().strip().splitlines()[-1]);print('invprio $v', d['value'])" || tail -3 gpurun_out/r2ip.err
done
