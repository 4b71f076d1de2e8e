#!/bin/bash
# final lines with peer-memory factor aggregation (default): multi-rank tests, N=4 and N=2 benches, N=1 bench
# (run with --gpus 4)
export PYTHONPATH=. SPD_WATCHDOG=900
timeout 900 python -m pytest tests/test_gpu_multi.py -m gpu -q -p no:cacheprovider > gpurun_out/r2p_multi_tests_p4.log 2>&1
echo "multi tests rc=$?"; tail -1 gpurun_out/r2p_multi_tests_p4.log
for N in 4 2; do
  TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
  for i in 1 2; do
    timeout 600 $TR --master-port $((29620 + RANDOM % 300)) bench.py --gpus $N --steps 20 --warmup 5 > gpurun_out/r2p_bench_n${N}_$i.json 2> gpurun_out/r2p_bench_n${N}_$i.err
    python -c "import json;d=json.loads(open('gpurun_out/r2p_bench_n${N}_$i.json').read().strip().splitlines()[-1]);print('n$N', d['value'], d['e2e']['value'], d['config']['factor_comm'], d['clocks']['reasons'])" || tail -3 gpurun_out/r2p_bench_n${N}_$i.err
  done
done
CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py > gpurun_out/r2p_bench_n1.json 2> gpurun_out/r2p_bench_n1.err
python -c "import json;d=json.loads(open('gpurun_out/r2p_bench_n1.json').read().strip().splitlines()[-1]);print('n1', d['value'], d['e2e']['value'], d['clocks']['reasons'])"
