#!/bin/bash
# N=4 env knobs with peer aggregation: gradient bucket share, early-G fractions (run with --gpus 4)
export PYTHONPATH=.
run() {  # tag env...
  tag=$1; shift
  TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
  env "$@" timeout 300 $TR --master-port $((29620 + RANDOM % 300)) bench.py --gpus 4 --steps 20 --warmup 5 > gpurun_out/k4_$tag.json 2> gpurun_out/k4_$tag.err
  python -c "import json;d=json.loads(open('gpurun_out/k4_$tag.json').read().strip().splitlines()[-1]);print('$tag', d['value'], d['e2e']['value'])" || tail -3 gpurun_out/k4_$tag.err
}
for r in a b; do
  run base_$r X=1
  run bucket95_$r SPDKFAC_GRAD_BUCKET=0.95
  run bucket80_$r SPDKFAC_GRAD_BUCKET=0.8
done
