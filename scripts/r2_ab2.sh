#!/bin/bash
# bench A/B (diagnostic): pairs on / off for the inverse update
export PYTHONPATH=.
for pr in 1 0; do
  SPDKFAC_UPDATE_PAIRS=$pr timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/ab_pairs$pr.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/ab_pairs$pr.json').read().strip().splitlines()[-1]);print('pairs=$pr', d['value'], {k:(v['kernel_ms_per_step'], v['frac']) for k,v in d['roofline_kernels'].items()})"
done
