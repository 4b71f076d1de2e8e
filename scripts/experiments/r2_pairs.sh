#!/bin/bash
# CTA-pair inverse update: correctness (inverse tests, pairs on) and isolated timing + bench, on / off.
export PYTHONPATH=. SPD_WATCHDOG=0
SPDKFAC_UPDATE_PAIRS=1 timeout 600 python -m pytest tests/test_gpu_linalg.py tests/test_gpu_production_paths.py -m gpu -q -p no:cacheprovider -k "inverse or nonpd" 2>&1 | tail -2
for pr in 1 0; do
  SPDKFAC_UPDATE_PAIRS=$pr timeout 300 python scripts/bench_inverse.py > gpurun_out/inv_pairs$pr.json 2>&1
  python -c "import json;d=json.load(open('gpurun_out/inv_pairs$pr.json'));print('pairs=$pr', {k:(d[k]['ms_total'], d[k]['cats'].get('inv_update',{}).get('ms'), d[k]['cats'].get('inv_update',{}).get('launches')) for k in ('d4608','d1024x8','resnet50_all108')})" || tail -5 gpurun_out/inv_pairs$pr.json
  SPDKFAC_UPDATE_PAIRS=$pr timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/ab_pairs$pr.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/ab_pairs$pr.json').read().strip().splitlines()[-1]);print('bench pairs=$pr', d['value'], d['roofline_kernels']['inv_update'])"
done
python scripts/prof_drivers.py inverse > /dev/null 2>&1 && SPDKFAC_UPDATE_PAIRS=1 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:tc3 --csv python scripts/prof_drivers.py inverse > gpurun_out/pairs_ncu1.csv 2>/dev/null
