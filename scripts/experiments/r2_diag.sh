#!/bin/bash
# U1 diagonal tiles first so the look-ahead pivot overlaps the rest of U1 (SPDKFAC_DIAG_FIRST=0: off)
export PYTHONPATH=. SPD_WATCHDOG=900
timeout 900 python -m pytest tests/test_gpu_linalg.py tests/test_gpu_production_paths.py -m gpu -q -p no:cacheprovider -k "inverse or damped or pivot or small" > gpurun_out/r2d_tests.log 2>&1
echo "tests rc=$?"; tail -1 gpurun_out/r2d_tests.log; grep -E "^E  |FAILED" gpurun_out/r2d_tests.log | head
for v in 1 0; do
  SPDKFAC_DIAG_FIRST=$v timeout 300 python scripts/bench_inverse.py > gpurun_out/r2d_inv_$v.json 2>&1
  python -c "
import json;d=json.load(open('gpurun_out/r2d_inv_$v.json'))
for k,v in d.items():
  if isinstance(v,dict): print('diag=$v', k, v['ms_total'])
"
done
timeout 900 python -m pytest tests/test_gpu_config_parity.py -m gpu -q -x -s -p no:cacheprovider -k "resnet50 or densenet" > gpurun_out/r2d_cfg.log 2>&1
echo "cfg rc=$?"; tail -1 gpurun_out/r2d_cfg.log
for v in 1 0 1 0; do
  SPDKFAC_DIAG_FIRST=$v timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/r2d_b.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/r2d_b.json').read().strip().splitlines()[-1]);print('bench diag=$v', d['value'])"
done
