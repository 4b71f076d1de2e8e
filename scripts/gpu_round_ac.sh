export SPD_WATCHDOG=250
timeout 600 python -m pytest tests/test_gpu_linalg.py -q -x -k "inverse" > gpurun_out/ac_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/ac_tests.log
timeout 300 python scripts/prof_kernels.py inverse 3 > gpurun_out/ac_inv.log 2>&1
timeout 300 python scripts/prof_kernels.py inverse_single 3 >> gpurun_out/ac_inv.log 2>&1
for i in 1 2; do
timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ac_new.log 2>&1
python -c "
import json
for l in open('gpurun_out/ac_new.log'):
    if l.startswith('{'):
        d=json.loads(l); print('new', d['value'])
" >> gpurun_out/ac_sum.log
done
