#!/bin/bash
# N=1 schedule knobs with the current kernels: early-G inversion groups, A launch groups
export PYTHONPATH=. SPD_WATCHDOG=900
run() {
  env $2 timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e $3 > gpurun_out/r2k_$1.json 2>gpurun_out/r2k_$1.err
  python -c "import json;d=json.loads(open('gpurun_out/r2k_$1.json').read().strip().splitlines()[-1]);print('$1', d['value'])" 2>/dev/null || echo "$1 failed"
}
run base "" ""
run f70 "" "--g-fractions 0.7,0.95,0.995"
run f80 "" "--g-fractions 0.8,0.97,0.997"
run f90 "" "--g-fractions 0.9,0.99,0.999"
run f2g "" "--g-fractions 0.85,0.99"
run ag1 "SPDKFAC_A_GROUPS=1" ""
run ag3 "SPDKFAC_A_GROUPS=3" ""
run base2 "" ""
run f70b "" "--g-fractions 0.7,0.95,0.995"
