#!/bin/bash
export PYTHONPATH=. SPD_WATCHDOG=900
timeout 900 python -m pytest tests/test_gpu_linalg.py tests/test_gpu_production_paths.py -m gpu -q -p no:cacheprovider -k "inverse or pivot or damped or small" > gpurun_out/r2_f16_tests.log 2>&1
echo "tests rc=$?"; tail -3 gpurun_out/r2_f16_tests.log; grep -E "^E  |FAILED" gpurun_out/r2_f16_tests.log | head
