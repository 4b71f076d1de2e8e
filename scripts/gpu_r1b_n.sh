export SPD_WATCHDOG=500
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/rn_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/rn_pytest.log
timeout 300 python scripts/prof_kernels.py inverse 5 > gpurun_out/rn_inv.log 2>&1
timeout 300 python scripts/prof_kernels.py inverse_single 3 > gpurun_out/rn_inv1.log 2>&1
run() { name=$1; shift; env "$@" timeout 300 python bench.py --no-cpu-baseline --no-e2e $BARGS > gpurun_out/rn_$name.log 2>&1; python -c "
import json
for l in open('gpurun_out/rn_$name.log'):
    if l.startswith('{'): print('$name', json.loads(l)['value'])
" >> gpurun_out/rn_sum.log; }
BARGS="" run base X=1
BARGS="" run tiles SPDKFAC_GRID=tiles
BARGS="--main-priority -1" run prio X=1
BARGS="--main-priority -1" run tiles_prio SPDKFAC_GRID=tiles
BARGS="" run cap120 SPDKFAC_MAX_CTAS=120
BARGS="--main-priority -1" run cap120_prio SPDKFAC_MAX_CTAS=120
