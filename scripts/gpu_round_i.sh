export SPD_WATCHDOG=120
timeout 900 python -m pytest tests/ -q -m gpu -x > gpurun_out/ri_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/ri_tests.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --timeline > gpurun_out/ri_n1.log 2>&1
python -c "
import json
for l in open('gpurun_out/ri_n1.log'):
    if l.startswith('{'):
        d=json.loads(l); print(d['value'], d['timeline_ms'])
" > gpurun_out/ri_sum.log
