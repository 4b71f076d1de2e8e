export SPD_WATCHDOG=120
timeout 900 python -m pytest tests/ -q -m gpu -x > gpurun_out/rn_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/rn_tests.log
timeout 300 python scripts/prof_kernels.py inverse 3 > gpurun_out/rn_prof.log 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --timeline > gpurun_out/rn_n1.log 2>&1
python -c "
import json
for l in open('gpurun_out/rn_n1.log'):
    if l.startswith('{'):
        d=json.loads(l); print(d['value'], d['e2e']['value'], d['timeline_ms'])
        print({k: v['ms_per_step'] for k, v in d['kernel_breakdown'].items() if isinstance(v, dict) and v['ms_per_step']})
" > gpurun_out/rn_sum.log
