#!/bin/bash
# TMA im2col SYRK (opt-in): parity (engine 3 vs staged im2col), production paths, config parity, bench A/B
export PYTHONPATH=. SPD_WATCHDOG=900
timeout 900 python -m pytest tests/test_gpu_production_paths.py tests/test_gpu_linalg.py -m gpu -q -p no:cacheprovider -k "im2col or conv or mixed or factor" > gpurun_out/r2_i2c_tests.log 2>&1
echo "tests rc=$?"; tail -1 gpurun_out/r2_i2c_tests.log; grep -E "^E  |FAILED" gpurun_out/r2_i2c_tests.log | head -12
SPDKFAC_IM2COL=1 timeout 900 python -m pytest tests/test_gpu_config_parity.py -m gpu -q -x -s -p no:cacheprovider > gpurun_out/r2_i2c_cfg.log 2>&1
echo "cfg (im2col on) rc=$?"; tail -1 gpurun_out/r2_i2c_cfg.log; grep worst gpurun_out/r2_i2c_cfg.log
for v in 1 0; do
SPDKFAC_IM2COL=$v timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/r2_i2c_bench$v.json 2>gpurun_out/r2_i2c_bench$v.err
python -c "import json;d=json.loads(open('gpurun_out/r2_i2c_bench$v.json').read().strip().splitlines()[-1]);print('bench i2c=$v', d['value'], {k:(v['kernel_ms_per_step'], v['frac']) for k,v in d['roofline_kernels'].items()})" || tail -5 gpurun_out/r2_i2c_bench$v.err
done
