export SPD_WATCHDOG=250
timeout 900 python -m pytest tests -m gpu -q -x --ignore=tests/test_gpu_multi.py > gpurun_out/v_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/v_tests.log
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --timeline > gpurun_out/v_bench.log 2>&1; echo "rc=$?" >> gpurun_out/v_bench.log
python -c "
import json
for l in open('gpurun_out/v_bench.log'):
    if l.startswith('{'):
        d=json.loads(l); print('n1', d['value'], d['e2e']['value'], d['roofline'], d['timeline_ms'])
        print({k: v['ms_per_step'] for k, v in d['kernel_breakdown'].items() if isinstance(v, dict) and v['ms_per_step']})
" > gpurun_out/v_sum.log
