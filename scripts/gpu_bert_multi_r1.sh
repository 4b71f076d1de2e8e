#!/bin/bash
# configs[4] at N=2/4: BERT-base linears, fused factor all-reduce + LBP-placed inverses.
mkdir -p gpurun_out
export SPD_WATCHDOG=300
for n in 2 4; do
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29900 + n)) bench.py --model bert_base_linears --gpus $n --steps 10 --warmup 3 > gpurun_out/bertm_n$n.json 2> gpurun_out/bertm_n$n.err
done
cut -c1-200 gpurun_out/bertm_n*.json; tail -3 gpurun_out/bertm_n4.err
