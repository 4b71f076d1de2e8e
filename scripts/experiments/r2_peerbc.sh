#!/bin/bash
# peer-memory inverse broadcast (SPDKFAC_PEER_BCAST, default on) vs NCCL broadcasts: parity + bench (--gpus N)
export PYTHONPATH=.
N=${1:-2}
timeout 420 python -m pytest tests/test_gpu_multi.py -m gpu -q -p no:cacheprovider > gpurun_out/peerbc_tests_$N.log 2>&1
echo "tests rc=$?"; tail -3 gpurun_out/peerbc_tests_$N.log
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29677"
for bc in 1 0 1 0; do
  SPDKFAC_PEER_BCAST=$bc timeout 300 $TR bench.py --gpus $N --steps 20 --warmup 5 > gpurun_out/peerbc${N}_$bc.json 2> gpurun_out/peerbc${N}_$bc.err
  echo "bc=$bc rc=$?"; python -c "import json;d=json.loads(open('gpurun_out/peerbc${N}_$bc.json').read().strip().splitlines()[-1]);print('bc=$bc', d['value'], d['ms_per_step'], d['e2e']['value'], d['config'].get('factor_comm'))"
done
