for args in "" "--inv-freq 1000" "--factor-freq 1000 --inv-freq 1000"; do
  timeout 600 python bench.py --steps 6 --warmup 3 --no-cpu-baseline --no-e2e $args > gpurun_out/da.log 2>&1
  python -c "
import json
for l in open('gpurun_out/da.log'):
    if l.startswith('{'):
        d=json.loads(l); print('ARGS [$args]', d['value'], d['host_wall_ms_per_step'], 'syrk', d['roofline']['kernel_ms_per_step'], d['roofline']['achieved'])
        print({k: v['ms_per_step'] for k, v in d['kernel_breakdown'].items() if isinstance(v, dict) and v['ms_per_step']})
" >> gpurun_out/da_sum.log
done
