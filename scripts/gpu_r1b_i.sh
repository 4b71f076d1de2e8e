export SPD_WATCHDOG=150
for i in 1 2; do
timeout 240 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $((29620 + i)) bench.py --gpus 4 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/ri_bench_n4_$i.log 2>&1; echo "rc=$?" >> gpurun_out/ri_bench_n4_$i.log
done
timeout 240 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29629 bench.py --gpus 4 --steps 10 --warmup 3 --no-cpu-baseline --mode eager > gpurun_out/ri_bench_n4_eager.log 2>&1; echo "rc=$?" >> gpurun_out/ri_bench_n4_eager.log
