export SPD_WATCHDOG=250
timeout 300 python -m pytest tests/test_gpu_linalg.py -x -q > gpurun_out/ah_tests.log 2>&1; echo "rc=$?" >> gpurun_out/ah_tests.log
grep -q "rc=0" gpurun_out/ah_tests.log || exit 1
timeout 300 python scripts/prof_kernels.py inverse 3 > gpurun_out/ah_inv.log 2>&1
(cd _ab_old && timeout 300 python scripts/prof_kernels.py inverse 3 > ../gpurun_out/ah_inv_old.log 2>&1)
timeout 300 python scripts/prof_kernels.py stage 5 > gpurun_out/ah_stage.log 2>&1
for i in 1 2; do
for w in old new; do
if [ $w = old ]; then cd _ab_old; else cd $GRAFT_REPO_ROOT; fi
timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > $GRAFT_REPO_ROOT/gpurun_out/ah.log 2>&1
cd $GRAFT_REPO_ROOT
python -c "
import json
for l in open('gpurun_out/ah.log'):
    if l.startswith('{'):
        d=json.loads(l); print('$w', d['value'], d['roofline']['kernel_ms_per_step'])
" >> gpurun_out/ah_sum.log
done
done
