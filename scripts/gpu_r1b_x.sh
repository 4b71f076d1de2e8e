export SPD_WATCHDOG=300
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/rx_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/rx_pytest.log
run() { name=$1; shift; env "$@" timeout 300 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/rx_$name.log 2>&1; python -c "
import json
for l in open('gpurun_out/rx_$name.log'):
    if l.startswith('{'): print('$name', json.loads(l)['value'])
" >> gpurun_out/rx_sum.log; }
run a2 SPDKFAC_A_GROUPS=2
run a1 SPDKFAC_A_GROUPS=1
run a4 SPDKFAC_A_GROUPS=4
run a8 SPDKFAC_A_GROUPS=8
run a2b SPDKFAC_A_GROUPS=2
run a4b SPDKFAC_A_GROUPS=4
