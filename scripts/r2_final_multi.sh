#!/bin/bash
# final N-GPU bench lines (default params, prefetched e2e) + multi-rank tests
N=${1:-2}
export PYTHONPATH=. SPD_WATCHDOG=900
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
timeout 900 python -m pytest tests/test_gpu_multi.py -m gpu -q -p no:cacheprovider > gpurun_out/r2f_multi_tests_p$N.log 2>&1
echo "multi tests rc=$?"; tail -1 gpurun_out/r2f_multi_tests_p$N.log
for i in 1 2; do
  timeout 600 $TR --master-port $((29620 + RANDOM % 300)) bench.py --gpus $N --steps 20 --warmup 5 > gpurun_out/r2f_bench_n${N}_$i.json 2> gpurun_out/r2f_bench_n${N}_$i.err
  python -c "import json;d=json.loads(open('gpurun_out/r2f_bench_n${N}_$i.json').read().strip().splitlines()[-1]);print('n$N', d['value'], d['e2e']['value'], d.get('placement_nct_tensors'))" || tail -3 gpurun_out/r2f_bench_n${N}_$i.err
done
