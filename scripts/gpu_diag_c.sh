python scripts/nvml_probe.py > gpurun_out/dd_sum.log 2>&1
for args in "--clocks off" "--clocks nvml" "--clocks smi" "--clocks nvml"; do
  timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e $args > gpurun_out/db.log 2>&1
  python -c "
import json
for l in open('gpurun_out/db.log'):
    if l.startswith('{'):
        d=json.loads(l); print('ARGS [$args]', d['value'], d['per_step_ms'], d['clocks'])
" >> gpurun_out/dd_sum.log
done
