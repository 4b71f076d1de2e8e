export SPD_WATCHDOG=120
timeout 300 python -m pytest tests/test_gpu_optimizer.py -q -x > gpurun_out/dc_tests.log 2>&1; echo "rc=$?" >> gpurun_out/dc_tests.log
for args in "" "--gc default" "" "--gc default"; do
  timeout 600 python bench.py --steps 8 --warmup 3 --no-cpu-baseline --no-e2e $args > gpurun_out/db.log 2>&1
  python -c "
import json
for l in open('gpurun_out/db.log'):
    if l.startswith('{'):
        d=json.loads(l); print('ARGS [$args]', d['value'], d['per_step_ms'])
" >> gpurun_out/dc_sum.log
done
