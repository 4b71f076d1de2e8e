export SPD_WATCHDOG=250
timeout 300 python scripts/prof_kernels.py stage 5 > gpurun_out/w_stage.log 2>&1; echo "rc=$?" >> gpurun_out/w_stage.log
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --timeline > gpurun_out/w_bench.log 2>&1; echo "rc=$?" >> gpurun_out/w_bench.log
python -c "
import json
for l in open('gpurun_out/w_bench.log'):
    if l.startswith('{'):
        d=json.loads(l); print('n1', d['value'], d['e2e']['value'], d['timeline_ms'])
        print({k: v['ms_per_step'] for k, v in d['kernel_breakdown'].items() if isinstance(v, dict) and v['ms_per_step']})
" > gpurun_out/w_sum.log
