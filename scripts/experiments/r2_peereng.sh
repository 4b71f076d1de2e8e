#!/bin/bash
# peer push engines: SM scatter vs copy engine, peer inverse broadcast on/off (run with --gpus N)
export PYTHONPATH=.
N=${1:-2}
timeout 420 python -m pytest tests/test_gpu_multi.py -m gpu -q -p no:cacheprovider -k peer > gpurun_out/peereng_tests_$N.log 2>&1
echo "tests rc=$?"; tail -2 gpurun_out/peereng_tests_$N.log
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29677"
for cfg in "sm 1" "sm 0" "ce 0" "sm 1" "sm 0" "ce 0"; do
  set -- $cfg
  SPDKFAC_PEER_ENGINE=$1 SPDKFAC_PEER_BCAST=$2 timeout 300 $TR bench.py --gpus $N --steps 20 --warmup 5 > gpurun_out/pe${N}_$1_$2.json 2> gpurun_out/pe${N}_$1_$2.err
  python -c "import json;d=json.loads(open('gpurun_out/pe${N}_$1_$2.json').read().strip().splitlines()[-1]);print('engine=$1 bcast=$2', d['value'], d['e2e']['value'])"
done
