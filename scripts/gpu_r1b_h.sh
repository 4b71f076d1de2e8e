export SPD_WATCHDOG=400
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q > gpurun_out/rh_multi.log 2>&1; echo "rc=$?" >> gpurun_out/rh_multi.log
for n in 2 4; do
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29600 + n)) bench.py --gpus $n --steps 10 --warmup 3 --trace gpurun_out/rh_trace_n$n.json > gpurun_out/rh_bench_n$n.log 2>&1; echo "rc=$?" >> gpurun_out/rh_bench_n$n.log
done
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus 4 --steps 10 --warmup 3 --balance dim_sq > gpurun_out/rh_bench_n4_dimsq.log 2>&1; echo "rc=$?" >> gpurun_out/rh_bench_n4_dimsq.log
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29612 bench.py --impl reference --gpus 2 --steps 2 --warmup 1 > gpurun_out/rh_ref_n2.log 2>&1; echo "rc=$?" >> gpurun_out/rh_ref_n2.log
