#!/bin/bash
# fp16 row-scaled preconditioning: parity, optimizer tests, config parity, bench A/B
export PYTHONPATH=. SPD_WATCHDOG=900
timeout 900 python -m pytest tests/test_gpu_linalg.py tests/test_gpu_production_paths.py tests/test_gpu_optimizer.py tests/test_gpu_reference_dropin.py -m gpu -q -p no:cacheprovider > gpurun_out/r2_prec_tests.log 2>&1
echo "tests rc=$?"; tail -1 gpurun_out/r2_prec_tests.log; grep -E "^E  |FAILED" gpurun_out/r2_prec_tests.log | head -12
timeout 900 python -m pytest tests/test_gpu_config_parity.py -m gpu -q -x -s -p no:cacheprovider > gpurun_out/r2_prec_cfg.log 2>&1
echo "cfg rc=$?"; tail -1 gpurun_out/r2_prec_cfg.log; grep worst gpurun_out/r2_prec_cfg.log
for v in 0 1; do
SPDKFAC_PRECOND_TF32=$v timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/r2_prec_bench$v.json 2>gpurun_out/r2_prec_bench$v.err
python -c "import json;d=json.loads(open('gpurun_out/r2_prec_bench$v.json').read().strip().splitlines()[-1]);print('bench tf32=$v', d['value'], {k:(v['kernel_ms_per_step'], v['frac']) for k,v in d['roofline_kernels'].items()})" || tail -5 gpurun_out/r2_prec_bench$v.err
done
