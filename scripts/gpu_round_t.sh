for args in "" "--main-priority -1" "--main-priority -3"; do
  timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e $args > gpurun_out/rt.log 2>&1
  python -c "
import json
for l in open('gpurun_out/rt.log'):
    if l.startswith('{'):
        d=json.loads(l); print('[$args]', d['value'])
" >> gpurun_out/rt_sum.log
done
for cap in 120 100; do
  SPDKFAC_MAX_CTAS=$cap timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --main-priority -1 > gpurun_out/rt.log 2>&1
  python -c "
import json
for l in open('gpurun_out/rt.log'):
    if l.startswith('{'):
        d=json.loads(l); print('[cap $cap prio -1]', d['value'])
" >> gpurun_out/rt_sum.log
done
