#!/bin/bash
export PYTHONPATH=. SPD_WATCHDOG=900
timeout 900 python -m pytest tests/test_gpu_linalg.py tests/test_gpu_production_paths.py tests/test_gpu_optimizer.py -m gpu -q -p no:cacheprovider > gpurun_out/r2r8_tests.log 2>&1
echo "tests rc=$?"; tail -1 gpurun_out/r2r8_tests.log; grep -E "^E  |FAILED" gpurun_out/r2r8_tests.log | head
timeout 900 python -m pytest tests/test_gpu_config_parity.py -m gpu -q -x -s -p no:cacheprovider > gpurun_out/r2r8_cfg.log 2>&1
echo "cfg rc=$?"; tail -1 gpurun_out/r2r8_cfg.log; grep worst gpurun_out/r2r8_cfg.log
for i in 1 2; do
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/r2r8_bench.json 2>gpurun_out/r2r8_bench.err
python -c "import json;d=json.loads(open('gpurun_out/r2r8_bench.json').read().strip().splitlines()[-1]);print('bench', d['value'], {k:(v['kernel_ms_per_step'], v['frac']) for k,v in d['roofline_kernels'].items()})"
done
python scripts/prof_drivers.py stage > /dev/null 2>&1 && ncu --clock-control none --kernel-name-base demangled -k "regex:stage_rows" -c 2 --metrics gpu__time_duration.sum,sm__inst_executed.avg.per_cycle_active python scripts/prof_drivers.py stage 2>&1 | grep -E "gpu__time|inst_exec" | head -4
