export SPD_WATCHDOG=250
timeout 400 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --trace gpurun_out/an_trace_n1.json > gpurun_out/an_n1.log 2>&1; echo "rc=$?" >> gpurun_out/an_n1.log
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29584 bench.py --gpus 2 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --trace gpurun_out/an_trace_n2.json > gpurun_out/an_n2.log 2>&1; echo "rc=$?" >> gpurun_out/an_n2.log
