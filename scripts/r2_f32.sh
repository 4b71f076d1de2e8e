#!/bin/bash
# fp32-rows SYRK (no staging for row layouts): parity tests, then bench A/B against staging.
export PYTHONPATH=. SPD_WATCHDOG=900
timeout 1500 python -m pytest tests/test_gpu_linalg.py tests/test_gpu_production_paths.py tests/test_gpu_optimizer.py tests/test_gpu_config_parity.py -m gpu -q -x -s -p no:cacheprovider -k "factor or syrk or stem or mixed or step or config or graphed or token or fixture" > gpurun_out/r2_f32_tests.log 2>&1
echo "tests rc=$?"; tail -3 gpurun_out/r2_f32_tests.log; grep -E "worst" gpurun_out/r2_f32_tests.log
for v in 1 0; do
  SPDKFAC_F32_ROWS=$v timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/ab_f32_$v.json 2>gpurun_out/ab_f32_$v.err
  python -c "import json;d=json.loads(open('gpurun_out/ab_f32_$v.json').read().strip().splitlines()[-1]);print('f32=$v', d['value'], {k:(v['kernel_ms_per_step'], v['frac']) for k,v in d['roofline_kernels'].items()})" || tail -5 gpurun_out/ab_f32_$v.err
done
