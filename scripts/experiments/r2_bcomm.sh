#!/bin/bash
# P > 1: inverse broadcasts on their own communicator/stream, issued as soon as each inverse group exists
N=${1:-2}
export PYTHONPATH=. SPD_WATCHDOG=600
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
timeout 900 python -m pytest tests/test_gpu_multi.py -m gpu -q -p no:cacheprovider > gpurun_out/r2bc_multi_tests_p$N.log 2>&1
echo "multi tests rc=$?"; tail -2 gpurun_out/r2bc_multi_tests_p$N.log; grep -E "^E  |FAILED" gpurun_out/r2bc_multi_tests_p$N.log | head
run() {
  env $2 timeout 420 $TR --master-port $((29620 + RANDOM % 300)) bench.py --gpus $N --steps 20 --warmup 5 $3 > gpurun_out/r2bc_$1.json 2> gpurun_out/r2bc_$1.err
  python -c "import json;d=json.loads(open('gpurun_out/r2bc_$1.json').read().strip().splitlines()[-1]);print('$1', d['value'], (d.get('e2e') or {}).get('value'))" || tail -3 gpurun_out/r2bc_$1.err
}
run sep "" ""
run one "SPDKFAC_BCAST_COMM=0" "--no-e2e"
run sep2 "" "--no-e2e"
run one2 "SPDKFAC_BCAST_COMM=0" "--no-e2e"
