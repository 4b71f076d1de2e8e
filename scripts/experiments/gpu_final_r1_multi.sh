#!/bin/bash
# Round-1 re-entry check at N=2/4: multi-rank GPU tests and bench lines.
mkdir -p gpurun_out
export SPD_WATCHDOG=250
timeout 600 python -m pytest tests/test_gpu_multi.py -q -x > gpurun_out/fm_multi.log 2>&1; echo "rc=$?" >> gpurun_out/fm_multi.log
for n in 2 4; do
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29800 + n)) bench.py --gpus $n --steps 20 --warmup 3 > gpurun_out/fm_bench_n$n.json 2> gpurun_out/fm_bench_n$n.err
done
tail -2 gpurun_out/fm_multi.log; cut -c1-200 gpurun_out/fm_bench_n*.json
