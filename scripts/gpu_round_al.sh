export SPD_WATCHDOG=250
timeout 300 python -m pytest tests/test_gpu_linalg.py -x -q -k inverse > gpurun_out/al_tests.log 2>&1; echo "rc=$?" >> gpurun_out/al_tests.log
grep -q "rc=0" gpurun_out/al_tests.log || exit 1
timeout 900 python -m pytest tests -m gpu -q -x --ignore=tests/test_gpu_multi.py > gpurun_out/al_tests2.log 2>&1; echo "rc=$?" >> gpurun_out/al_tests2.log
timeout 300 python scripts/prof_kernels.py inverse 3 > gpurun_out/al_inv.log 2>&1
timeout 300 python scripts/prof_kernels.py inverse_single 3 >> gpurun_out/al_inv.log 2>&1
for i in 1 2; do
for w in old new; do
if [ $w = old ]; then cd _ab_old; else cd $GRAFT_REPO_ROOT; fi
timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > $GRAFT_REPO_ROOT/gpurun_out/al.log 2>&1
cd $GRAFT_REPO_ROOT
python -c "
import json
for l in open('gpurun_out/al.log'):
    if l.startswith('{'):
        d=json.loads(l); print('$w', d['value'])
" >> gpurun_out/al_sum.log
done
done
