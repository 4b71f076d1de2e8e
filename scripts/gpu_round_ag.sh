export SPD_WATCHDOG=250
timeout 300 python -m pytest tests/test_gpu_linalg.py -x -q -k factor > gpurun_out/ag_tests.log 2>&1; echo "rc=$?" >> gpurun_out/ag_tests.log
grep -q "rc=0" gpurun_out/ag_tests.log || exit 1
timeout 600 python -m pytest tests -m gpu -q -x --ignore=tests/test_gpu_multi.py > gpurun_out/ag_tests2.log 2>&1; echo "rc=$?" >> gpurun_out/ag_tests2.log
timeout 300 python scripts/prof_kernels.py stage 5 > gpurun_out/ag_stage.log 2>&1
for i in 1 2; do
for w in old new; do
if [ $w = old ]; then cd _ab_old; else cd $GRAFT_REPO_ROOT; fi
timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > $GRAFT_REPO_ROOT/gpurun_out/ag.log 2>&1
cd $GRAFT_REPO_ROOT
python -c "
import json
for l in open('gpurun_out/ag.log'):
    if l.startswith('{'):
        d=json.loads(l); print('$w', d['value'], d['roofline']['kernel_ms_per_step'])
" >> gpurun_out/ag_sum.log
done
done
