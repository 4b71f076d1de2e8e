#!/bin/bash
# P=2 auto launch groups (inversion cuts with peer aggregation): multi-rank tests + bench (run with --gpus 2)
export PYTHONPATH=.
timeout 600 python -m pytest tests/test_gpu_multi.py -m gpu -q -p no:cacheprovider > gpurun_out/lg2_tests.log 2>&1
echo "tests rc=$?"; tail -3 gpurun_out/lg2_tests.log
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
for i in 1 2; do
  timeout 300 $TR --master-port $((29620 + RANDOM % 300)) bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/lg2_bench_$i.json 2> gpurun_out/lg2_bench_$i.err
  python -c "import json;d=json.loads(open('gpurun_out/lg2_bench_$i.json').read().strip().splitlines()[-1]);print('n2', d['value'], d['e2e']['value'], d['config']['fusion'])" || tail -3 gpurun_out/lg2_bench_$i.err
done
