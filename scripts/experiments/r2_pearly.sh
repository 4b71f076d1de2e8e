#!/bin/bash
# P > 1 early-group preconditioning in step() (SPDKFAC_EARLY_PRECOND): multi-rank parity + bench A/B (--gpus 4)
export PYTHONPATH=.
timeout 900 python -m pytest tests/test_gpu_multi.py -m gpu -q -p no:cacheprovider > gpurun_out/pe_tests.log 2>&1
echo "tests rc=$?"; tail -3 gpurun_out/pe_tests.log
run() {  # N early tag
  TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $1 --master-addr 127.0.0.1"
  SPDKFAC_EARLY_PRECOND=$2 timeout 300 $TR --master-port $((29620 + RANDOM % 300)) bench.py --gpus $1 --steps 20 --warmup 5 > gpurun_out/pe_$3.json 2> gpurun_out/pe_$3.err
  python -c "import json;d=json.loads(open('gpurun_out/pe_$3.json').read().strip().splitlines()[-1]);print('$3', d['value'], d['e2e']['value'])" || tail -3 gpurun_out/pe_$3.err
}
run 4 1 n4_on; run 4 0 n4_off; run 2 1 n2_on; run 2 0 n2_off; run 4 1 n4_on_b; run 4 0 n4_off_b; run 2 1 n2_on_b; run 2 0 n2_off_b
