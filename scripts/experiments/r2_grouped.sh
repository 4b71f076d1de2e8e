#!/bin/bash
# P > 1 grouped preconditioning (early groups beside the tail inversion) vs one plan at the end
N=${1:-2}
export PYTHONPATH=. SPD_WATCHDOG=900
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
timeout 1200 python -m pytest tests/test_gpu_multi.py -m gpu -q -p no:cacheprovider > gpurun_out/r2g_multi_tests_p$N.log 2>&1
echo "multi tests rc=$?"; tail -2 gpurun_out/r2g_multi_tests_p$N.log; grep -E "^E  |FAILED" gpurun_out/r2g_multi_tests_p$N.log | head
run() {
  env $2 timeout 900 $TR --master-port $((29620 + RANDOM % 300)) bench.py --gpus $N --steps 20 --warmup 5 $3 > gpurun_out/r2g_$1.json 2> gpurun_out/r2g_$1.err
  python -c "import json;d=json.loads(open('gpurun_out/r2g_$1.json').read().strip().splitlines()[-1]);print('$1', d['value'], (d.get('e2e') or {}).get('value'))" || tail -3 gpurun_out/r2g_$1.err
}
run grouped "" ""
run single "SPDKFAC_GROUPED_PRECOND=0" "--no-e2e"
run grouped2 "" "--no-e2e"
run single2 "SPDKFAC_GROUPED_PRECOND=0" "--no-e2e"
