#!/bin/bash
# N=1: cap every persistent tile-engine grid (SPDKFAC_MAX_CTAS) to leave SMs to cuDNN / the inversion chains
export PYTHONPATH=.
for c in 0 140 128 0 140 128; do
  if [ $c = 0 ]; then unset SPDKFAC_MAX_CTAS; else export SPDKFAC_MAX_CTAS=$c; fi
  timeout 300 python bench.py --steps 20 --warmup 5 > gpurun_out/mc_$c.json 2> gpurun_out/mc_$c.err
  python -c "import json;d=json.loads(open('gpurun_out/mc_$c.json').read().strip().splitlines()[-1]);print('max_ctas=$c', d['value'], d['e2e']['value'], d['clocks']['reasons'])"
done
