#!/bin/bash
# peer-memory factor aggregation at 4 ranks: parity vs NCCL reduce and bench A/B (run with --gpus 4)
export PYTHONPATH=.
timeout 420 python -m pytest tests/test_gpu_multi.py -m gpu -q -k "peer" -p no:cacheprovider -s > gpurun_out/peer4_tests.log 2>&1
echo "tests rc=$?"; tail -c 1500 gpurun_out/peer4_tests.log
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29677"
for fc in peer reduce peer reduce; do
  timeout 300 $TR bench.py --gpus 4 --steps 20 --warmup 5 --factor-comm $fc > gpurun_out/peer4_bench_$fc.json 2> gpurun_out/peer4_bench_$fc.err
  echo "$fc rc=$?"; python -c "import json;d=json.loads(open('gpurun_out/peer4_bench_$fc.json').read().strip().splitlines()[-1]);print('$fc', d['value'], d['ms_per_step'], d['e2e']['value'], d['config'].get('factor_comm'))"
done
