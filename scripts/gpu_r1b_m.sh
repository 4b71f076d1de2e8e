export SPD_WATCHDOG=200
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q > gpurun_out/rm_multi.log 2>&1; echo "rc=$?" >> gpurun_out/rm_multi.log
timeout 240 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29701 bench.py --gpus 2 --steps 10 --warmup 3 --trace gpurun_out/rm_trace_n2.json > gpurun_out/rm_bench_n2_trace.log 2>&1; echo "rc=$?" >> gpurun_out/rm_bench_n2_trace.log
for i in 1 2; do
for n in 2 4; do
timeout 240 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29710 + 10*i + n)) bench.py --gpus $n --steps 10 --warmup 3 > gpurun_out/rm_bench_n${n}_$i.log 2>&1; echo "rc=$?" >> gpurun_out/rm_bench_n${n}_$i.log
done
done
