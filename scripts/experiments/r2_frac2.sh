#!/bin/bash
# P > 1: early G inversion-group fractions
N=${1:-2}
export PYTHONPATH=. SPD_WATCHDOG=600
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
run() {
  timeout 300 $TR --master-port $((29620 + RANDOM % 300)) bench.py --gpus $N --steps 20 --warmup 5 --no-e2e $2 > gpurun_out/r2fr_$1.json 2> gpurun_out/r2fr_$1.err
  python -c "import json;d=json.loads(open('gpurun_out/r2fr_$1.json').read().strip().splitlines()[-1]);print('$1', d['value'])" 2>/dev/null || echo "$1 failed"
}
run base ""
run f1 "--g-fractions 0.7,0.9,0.98"
run f2 "--g-fractions 0.5,0.8,0.95"
run f3 "--g-fractions 0.6,0.85,0.95,0.99"
run f4 "--g-fractions 0.8,0.95"
run base2 ""
run f1b "--g-fractions 0.7,0.9,0.98"
