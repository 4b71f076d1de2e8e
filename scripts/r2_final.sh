#!/bin/bash
# full -m gpu suite, default bench line (N=1), reference arm
export PYTHONPATH=. SPD_WATCHDOG=900
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2_final_tests.log 2>&1
echo "tests rc=$?"; tail -2 gpurun_out/r2_final_tests.log; grep -E "FAILED" gpurun_out/r2_final_tests.log | head
timeout 900 python bench.py > gpurun_out/r2_final_bench.json 2>gpurun_out/r2_final_bench.err
echo "bench rc=$?"; python -c "import json;d=json.loads(open('gpurun_out/r2_final_bench.json').read().strip().splitlines()[-1]);print('bench', d['value'], d['e2e'], d['roofline']['kernel'], d['roofline']['frac'], d.get('iteration_roofline',{}).get('frac') if d.get('iteration_roofline') else None, d['clocks'])"
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_final_smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/r2_final_smoke.log
