#!/bin/bash
# fp16-plane inverse panel / update: parity, isolated inverse timing f16 vs tf32, config parity, bench
export PYTHONPATH=. SPD_WATCHDOG=900
timeout 900 python -m pytest tests/test_gpu_linalg.py tests/test_gpu_production_paths.py -m gpu -q -x -s -p no:cacheprovider -k "inverse or pivot or damped or small" > gpurun_out/r2_f16_tests.log 2>&1
echo "tests rc=$?"; tail -3 gpurun_out/r2_f16_tests.log; grep -E "d=4608|d=2048" gpurun_out/r2_f16_tests.log
for v in 0 1; do
  SPDKFAC_INV_TF32=$v timeout 300 python scripts/bench_inverse.py > gpurun_out/r2_inv_iso_tf32$v.json 2>&1; echo "inv tf32=$v rc=$?"
  python -c "
import json;d=json.load(open('gpurun_out/r2_inv_iso_tf32$v.json'))
for k,v in d.items():
  if isinstance(v,dict): print('tf32=$v', k, v['ms_total'], {c:(x['ms'],x['launches'],x['us_per_launch']) for c,x in v['cats'].items()})
" || tail -5 gpurun_out/r2_inv_iso_tf32$v.json
done
timeout 900 python -m pytest tests/test_gpu_config_parity.py -m gpu -q -x -s -p no:cacheprovider > gpurun_out/r2_f16_cfg.log 2>&1
echo "cfg rc=$?"; tail -2 gpurun_out/r2_f16_cfg.log; grep worst gpurun_out/r2_f16_cfg.log
for v in 0 1; do
SPDKFAC_INV_TF32=$v timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/r2_f16_bench$v.json 2>gpurun_out/r2_f16_bench$v.err
python -c "import json;d=json.loads(open('gpurun_out/r2_f16_bench$v.json').read().strip().splitlines()[-1]);print('bench tf32=$v', d['value'], {k:(v['kernel_ms_per_step'], v['frac']) for k,v in d['roofline_kernels'].items()})" || tail -5 gpurun_out/r2_f16_bench$v.err
done
