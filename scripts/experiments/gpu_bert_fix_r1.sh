#!/bin/bash
# Large pack-batch fix: regression test + configs[4] at N=2/4 + the ResNet-50 multi-rank tests.
mkdir -p gpurun_out
export SPD_WATCHDOG=300
timeout 300 python -m pytest tests/test_gpu_linalg.py -q -x -k pack > gpurun_out/bf_pack.log 2>&1; echo "rc=$?" >> gpurun_out/bf_pack.log
for n in 2 4; do
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29900 + n)) bench.py --model bert_base_linears --gpus $n --steps 10 --warmup 3 > gpurun_out/bertm_n$n.json 2> gpurun_out/bertm_n$n.err
done
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29952 bench.py --gpus 2 --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bf_r50_n2.json 2> gpurun_out/bf_r50_n2.err
tail -2 gpurun_out/bf_pack.log; cut -c1-200 gpurun_out/bertm_n*.json gpurun_out/bf_r50_n2.json
