#!/bin/bash
export PYTHONPATH=. SPD_WATCHDOG=900
timeout 900 python -m pytest tests/test_gpu_linalg.py tests/test_gpu_production_paths.py tests/test_gpu_optimizer.py -m gpu -q -p no:cacheprovider > gpurun_out/r2_prec2_tests.log 2>&1
echo "tests rc=$?"; tail -1 gpurun_out/r2_prec2_tests.log; grep -E "^E  |FAILED" gpurun_out/r2_prec2_tests.log | head -12
timeout 900 python -m pytest tests/test_gpu_config_parity.py -m gpu -q -x -s -p no:cacheprovider > gpurun_out/r2_prec2_cfg.log 2>&1
echo "cfg rc=$?"; tail -1 gpurun_out/r2_prec2_cfg.log; grep worst gpurun_out/r2_prec2_cfg.log
