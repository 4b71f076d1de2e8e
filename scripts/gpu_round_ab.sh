export SPD_WATCHDOG=250
timeout 900 python -m pytest tests -m gpu -q -x --ignore=tests/test_gpu_multi.py > gpurun_out/ab_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/ab_tests.log
timeout 300 python scripts/prof_kernels.py stage 5 > gpurun_out/ab_stage.log 2>&1
for i in 1 2; do
(cd _ab_old && timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > ../gpurun_out/ab_old.log 2>&1)
timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab_new.log 2>&1
for w in old new; do python -c "
import json
for l in open('gpurun_out/ab_$w.log'):
    if l.startswith('{'):
        d=json.loads(l); print('$w', d['value'])
" >> gpurun_out/ab_sum.log; done
done
