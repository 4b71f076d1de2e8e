#!/bin/bash
# inversion-cut launch groups with more A groups (SPDKFAC_A_GROUPS) at N=4 / N=2 (run with --gpus 4)
export PYTHONPATH=.
run() {  # N launch_groups a_groups tag
  TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $1 --master-addr 127.0.0.1"
  SPDKFAC_A_GROUPS=$3 timeout 300 $TR --master-port $((29620 + RANDOM % 300)) bench.py --gpus $1 --steps 20 --warmup 5 --launch-groups $2 > gpurun_out/ag_$4.json 2> gpurun_out/ag_$4.err
  python -c "import json;d=json.loads(open('gpurun_out/ag_$4.json').read().strip().splitlines()[-1]);print('$4', d['value'], d['e2e']['value'])" || tail -3 gpurun_out/ag_$4.err
}
run 4 inversion 8 n4_inv8; run 4 inversion 16 n4_inv16; run 4 fusion 2 n4_fusion
run 2 inversion 4 n2_inv4; run 2 inversion 2 n2_inv2
run 4 inversion 8 n4_inv8b; run 4 fusion 2 n4_fusionb
