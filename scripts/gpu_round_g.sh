export SPD_WATCHDOG=120
timeout 180 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/rg_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/rg_smoke.log
timeout 900 python -m pytest tests/ -q -m gpu -x > gpurun_out/rg_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/rg_tests.log
for args in "" "--memory-format nchw" "--optimizer sgd" "--optimizer sgd --mode eager --memory-format nchw"; do
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline $args > gpurun_out/rg_n1.log 2>&1
python -c "
import json
for l in open('gpurun_out/rg_n1.log'):
    if l.startswith('{'):
        d=json.loads(l); print('[$args]', d['value'], d['per_step_ms'], d['e2e'])
        print({k: v['ms_per_step'] for k, v in d['kernel_breakdown'].items() if isinstance(v, dict) and v['ms_per_step']})
" >> gpurun_out/rg_sum.log; tail -2 gpurun_out/rg_n1.log | cut -c1-300 >> gpurun_out/rg_sum.log
done
