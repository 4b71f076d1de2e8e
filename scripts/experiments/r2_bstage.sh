#!/bin/bash
# deferred batched row staging (one launch per group compute) vs per-member staging
export PYTHONPATH=. SPD_WATCHDOG=900
timeout 900 python -m pytest tests/test_gpu_linalg.py tests/test_gpu_production_paths.py tests/test_gpu_optimizer.py -m gpu -q -p no:cacheprovider > gpurun_out/r2bs_tests.log 2>&1
echo "tests rc=$?"; tail -1 gpurun_out/r2bs_tests.log; grep -E "^E  |FAILED" gpurun_out/r2bs_tests.log | head
timeout 900 python -m pytest tests/test_gpu_config_parity.py -m gpu -q -x -s -p no:cacheprovider > gpurun_out/r2bs_cfg.log 2>&1
echo "cfg rc=$?"; tail -1 gpurun_out/r2bs_cfg.log; grep worst gpurun_out/r2bs_cfg.log
for v in 1 0 1 0; do
  SPDKFAC_BATCH_STAGE=$v timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/r2bs_b.json 2>gpurun_out/r2bs_b.err
  python -c "import json;d=json.loads(open('gpurun_out/r2bs_b.json').read().strip().splitlines()[-1]);print('bench batch=$v', d['value'], d['roofline_kernels']['factor_stage']['kernel_ms_per_step'], d['roofline_kernels']['factor_syrk']['kernel_ms_per_step'])" || tail -3 gpurun_out/r2bs_b.err
done
