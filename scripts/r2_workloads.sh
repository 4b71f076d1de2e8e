#!/bin/bash
# BASELINE configs[3] / [4] and the BERT-base linears with the current kernels (N=1)
export PYTHONPATH=. SPD_WATCHDOG=900
for cfg in "bert_base_linears 32"; do
  set -- $cfg
  timeout 900 python bench.py --model $1 --batch $2 --steps 10 --warmup 4 --no-cpu-baseline > gpurun_out/r2w_$1.json 2> gpurun_out/r2w_$1.err
  python -c "import json;d=json.loads(open('gpurun_out/r2w_$1.json').read().strip().splitlines()[-1]);print('$1', d['value'], (d.get('e2e') or {}).get('value'), d['roofline']['kernel'][:40], d['roofline']['frac'])" || tail -3 gpurun_out/r2w_$1.err
done
