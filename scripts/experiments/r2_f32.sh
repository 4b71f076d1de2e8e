#!/bin/bash
# fp32-rows SYRK (no staging for row layouts with d <= 256): parity tests, bench A/B, pivot timing.
export PYTHONPATH=. SPD_WATCHDOG=900
timeout 1500 python -m pytest tests/test_gpu_linalg.py tests/test_gpu_production_paths.py tests/test_gpu_optimizer.py tests/test_gpu_config_parity.py -m gpu -q -x -s -p no:cacheprovider > gpurun_out/r2_f32_tests.log 2>&1
echo "tests rc=$?"; tail -3 gpurun_out/r2_f32_tests.log; grep -E "worst" gpurun_out/r2_f32_tests.log
for v in 2 0 1; do
  SPDKFAC_F32_ROWS=$v timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/ab_f32_$v.json 2>gpurun_out/ab_f32_$v.err
  python -c "import json;d=json.loads(open('gpurun_out/ab_f32_$v.json').read().strip().splitlines()[-1]);print('f32=$v', d['value'], {k:(v['kernel_ms_per_step'], v['frac']) for k,v in d['roofline_kernels'].items()})" || tail -5 gpurun_out/ab_f32_$v.err
done
timeout 600 python scripts/bench_inverse.py > gpurun_out/r2_inv_iso.json 2>&1; echo "inv rc=$?"; head -c 1500 gpurun_out/r2_inv_iso.json
