#!/bin/bash
# N=1: cap the preconditioning GEMM grid so the tail inversion chain co-runs (SPDKFAC_PRECOND_CTAS)
export PYTHONPATH=.
for c in 0 136 120 0 136 120; do
  SPDKFAC_PRECOND_CTAS=$c timeout 300 python bench.py --steps 20 --warmup 5 > gpurun_out/pc_$c.json 2> gpurun_out/pc_$c.err
  python -c "import json;d=json.loads(open('gpurun_out/pc_$c.json').read().strip().splitlines()[-1]);print('ctas=$c', d['value'], d['e2e']['value'], d['clocks']['reasons'])"
done
