#!/bin/bash
export PYTHONPATH=. SPD_WATCHDOG=900
for p in 0 -1 -5 0 -1; do
  timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --main-priority $p > gpurun_out/r2p_$p.json 2>gpurun_out/r2p_$p.err
  python -c "import json;d=json.loads(open('gpurun_out/r2p_$p.json').read().strip().splitlines()[-1]);print('prio $p', d['value'])" || tail -3 gpurun_out/r2p_$p.err
done
