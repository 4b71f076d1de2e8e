#!/bin/bash
export PYTHONPATH=. SPD_WATCHDOG=900
timeout 900 python -m pytest tests/test_gpu_optimizer.py -m gpu -q -p no:cacheprovider -k "graphed or prefetch" > gpurun_out/r2_pf_tests.log 2>&1
echo "tests rc=$?"; tail -1 gpurun_out/r2_pf_tests.log; grep -E "^E  |FAILED" gpurun_out/r2_pf_tests.log | head
timeout 900 python bench.py > gpurun_out/r2_pf_bench.json 2>gpurun_out/r2_pf_bench.err
echo "bench rc=$?"; python -c "import json;d=json.loads(open('gpurun_out/r2_pf_bench.json').read().strip().splitlines()[-1]);print('bench', d['value'], d['e2e'], d['cpu_baseline'], d['clocks'])"
