#!/bin/bash
# CTA-pair update engine over fp16 planes (SPDKFAC_UPDATE_PAIRS=1) vs single-CTA tiles
export PYTHONPATH=. SPD_WATCHDOG=900
for v in 1 0; do
SPDKFAC_UPDATE_PAIRS=$v timeout 900 python -m pytest tests/test_gpu_linalg.py tests/test_gpu_production_paths.py -m gpu -q -p no:cacheprovider -k "inverse or damped" > gpurun_out/r2p16_tests_$v.log 2>&1
echo "tests pairs=$v rc=$?"; tail -1 gpurun_out/r2p16_tests_$v.log; grep -E "^E  |FAILED" gpurun_out/r2p16_tests_$v.log | head -5
done
for v in 1 0; do
  SPDKFAC_UPDATE_PAIRS=$v timeout 300 python scripts/bench_inverse.py > gpurun_out/r2p16_inv_$v.json 2>&1
  python -c "
import json;d=json.load(open('gpurun_out/r2p16_inv_$v.json'))
for k,v in d.items():
  if isinstance(v,dict): print('pairs=$v', k, v['ms_total'], v['cats'].get('inv_update'))
"
done
SPDKFAC_UPDATE_PAIRS=1 timeout 900 python -m pytest tests/test_gpu_config_parity.py -m gpu -q -x -s -p no:cacheprovider -k "resnet50" > gpurun_out/r2p16_cfg.log 2>&1
echo "cfg rc=$?"; tail -1 gpurun_out/r2p16_cfg.log
for v in 1 0 1 0; do
  SPDKFAC_UPDATE_PAIRS=$v timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/r2p16_b.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/r2p16_b.json').read().strip().splitlines()[-1]);print('bench pairs=$v', d['value'])"
done
