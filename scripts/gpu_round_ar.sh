export SPD_WATCHDOG=250
for n in 2 4; do
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29800 + n)) bench.py --gpus $n --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --trace gpurun_out/ar_trace_n$n.json > gpurun_out/ar_n$n.log 2>&1
done
