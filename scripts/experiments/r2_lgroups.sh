#!/bin/bash
# P > 1 with peer aggregation: SYRK/aggregation launch groups = fusion plan vs inversion-group cuts (run with --gpus 4)
export PYTHONPATH=.
for N in 4 2; do
  TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
  for lg in inversion fusion inversion fusion; do
    timeout 300 $TR --master-port $((29620 + RANDOM % 300)) bench.py --gpus $N --steps 20 --warmup 5 --launch-groups $lg > gpurun_out/lg_n${N}_$lg.json 2> gpurun_out/lg_n${N}_$lg.err
    python -c "import json;d=json.loads(open('gpurun_out/lg_n${N}_$lg.json').read().strip().splitlines()[-1]);print('n$N $lg', d['value'], d['e2e']['value'])" || tail -3 gpurun_out/lg_n${N}_$lg.err
  done
done
