export SPD_WATCHDOG=120
timeout 600 python -m pytest tests/test_gpu_optimizer.py -q -x > gpurun_out/re_tests.log 2>&1; echo "rc=$?" >> gpurun_out/re_tests.log
for args in "" "--mode eager"; do
  timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline $args > gpurun_out/re_bench.log 2>&1
  python -c "
import json
for l in open('gpurun_out/re_bench.log'):
    if l.startswith('{'):
        d=json.loads(l); print('ARGS [$args]', d['value'], d['per_step_ms'], d['e2e'], d['gpu_launches'], d['roofline']['kernel_ms_per_step'], d['roofline']['achieved'], d['allocator_in_region'])
" >> gpurun_out/re_sum.log
  tail -3 gpurun_out/re_bench.log | cut -c1-400 >> gpurun_out/re_sum.log
done
