export SPD_WATCHDOG=500
timeout 900 python -m pytest tests/test_gpu_linalg.py -x -q > gpurun_out/ro_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/ro_pytest.log
run() { name=$1; shift; env "$@" timeout 300 python bench.py --no-cpu-baseline --no-e2e $BARGS > gpurun_out/ro_$name.log 2>&1; python -c "
import json
for l in open('gpurun_out/ro_$name.log'):
    if l.startswith('{'): print('$name', json.loads(l)['value'])
" >> gpurun_out/ro_sum.log; }
BARGS="" run pc0 SPDKFAC_PANEL_CTAS=0
BARGS="" run pc32 SPDKFAC_PANEL_CTAS=32
BARGS="" run pc16 SPDKFAC_PANEL_CTAS=16
BARGS="" run pc64 SPDKFAC_PANEL_CTAS=64
BARGS="" run pc32b SPDKFAC_PANEL_CTAS=32
BARGS="" run pc0b SPDKFAC_PANEL_CTAS=0
SPDKFAC_PANEL_CTAS=0 timeout 300 python scripts/prof_kernels.py inverse 5 > gpurun_out/ro_inv_pc0.log 2>&1
SPDKFAC_PANEL_CTAS=32 timeout 300 python scripts/prof_kernels.py inverse 5 > gpurun_out/ro_inv_pc32.log 2>&1
