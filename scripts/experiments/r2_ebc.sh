#!/bin/bash
# P > 1: early G-group broadcasts right after each inversion + grouped preconditioning (SPDKFAC_EARLY_BCAST=1)
N=${1:-2}
export PYTHONPATH=. SPD_WATCHDOG=600
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
SPDKFAC_EARLY_BCAST=1 timeout 700 python -m pytest tests/test_gpu_multi.py -m gpu -q -p no:cacheprovider > gpurun_out/r2ebc_tests_p$N.log 2>&1
echo "multi tests (early bcast) rc=$?"; tail -2 gpurun_out/r2ebc_tests_p$N.log; grep -E "^E  |FAILED" gpurun_out/r2ebc_tests_p$N.log | head
run() {
  env $2 timeout 400 $TR --master-port $((29620 + RANDOM % 300)) bench.py --gpus $N --steps 20 --warmup 5 --no-e2e > gpurun_out/r2ebc_$1.json 2> gpurun_out/r2ebc_$1.err
  python -c "import json;d=json.loads(open('gpurun_out/r2ebc_$1.json').read().strip().splitlines()[-1]);print('$1', d['value'])" 2>/dev/null || echo "$1 failed"
}
run ebc "SPDKFAC_EARLY_BCAST=1"
run base ""
run ebc2 "SPDKFAC_EARLY_BCAST=1"
run base2 ""
