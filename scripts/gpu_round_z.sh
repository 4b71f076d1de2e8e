export SPD_WATCHDOG=250
timeout 300 python -m pytest tests/test_gpu_linalg.py -x -q -k factor > gpurun_out/z_tests.log 2>&1; echo "rc=$?" >> gpurun_out/z_tests.log
timeout 300 python scripts/prof_kernels.py stage 5 > gpurun_out/z_stage.log 2>&1
for i in 1 2; do
(cd _ab_old && timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e --timeline > ../gpurun_out/z_old.log 2>&1)
timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e --timeline > gpurun_out/z_new.log 2>&1
for w in old new; do python -c "
import json
for l in open('gpurun_out/z_$w.log'):
    if l.startswith('{'):
        d=json.loads(l); print('$w', d['value'], d['timeline_ms'])
" >> gpurun_out/z_sum.log; done
done
