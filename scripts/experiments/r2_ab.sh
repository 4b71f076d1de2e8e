#!/bin/bash
# A/B of bench variants on one box (diagnostic): default (probes on the roofline categories),
# --stats-off, SPDKFAC_PIVOT=tc.  Each: 20 timed steps after 5 warm-up, no CPU leg.
export PYTHONPATH=.
for v in "default|" "statsoff|--stats-off" "pivtc|"; do
  name=${v%%|*}; flags=${v#*|}
  if [ "$name" = pivtc ]; then export SPDKFAC_PIVOT=tc; else unset SPDKFAC_PIVOT; fi
  timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e $flags > gpurun_out/ab_$name.json 2>gpurun_out/ab_$name.err
  python -c "import json;d=json.loads(open('gpurun_out/ab_$name.json').read().strip().splitlines()[-1]);print('$name', d['value'], d['per_step_ms'][:4], {k:(v['kernel_ms_per_step'], v['frac']) for k,v in (d.get('roofline_kernels') or {}).items()})"
done
