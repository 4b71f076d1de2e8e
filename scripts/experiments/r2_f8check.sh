#!/bin/bash
export PYTHONPATH=. SPD_WATCHDOG=900
timeout 900 python -m pytest tests/test_gpu_config_parity.py tests/test_gpu_production_paths.py -m gpu -q -x -s -p no:cacheprovider > gpurun_out/r2_f8_cfg.log 2>&1
echo "cfg rc=$?"; tail -1 gpurun_out/r2_f8_cfg.log; grep -E "worst|d=4608|d=2048" gpurun_out/r2_f8_cfg.log
timeout 600 python bench.py --steps 20 --warmup 5 --trace gpurun_out/r2_trace > gpurun_out/r2_f8_trace.json 2>gpurun_out/r2_f8_trace.err
echo "trace rc=$?"; ls gpurun_out/r2_trace* 2>/dev/null; tail -2 gpurun_out/r2_f8_trace.err
