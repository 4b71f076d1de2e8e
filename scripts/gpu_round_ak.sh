export SPD_WATCHDOG=250
timeout 900 python -m pytest tests -m gpu -q -x --ignore=tests/test_gpu_multi.py > gpurun_out/ak_tests.log 2>&1; echo "rc=$?" >> gpurun_out/ak_tests.log
timeout 400 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --trace gpurun_out/ak_trace_n1.json > gpurun_out/ak_n1.log 2>&1; echo "rc=$?" >> gpurun_out/ak_n1.log
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29582 bench.py --gpus 2 --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ak_n2.log 2>&1; echo "rc=$?" >> gpurun_out/ak_n2.log
timeout 600 python -m pytest tests/test_gpu_multi.py -q -x > gpurun_out/ak_multi.log 2>&1; echo "rc=$?" >> gpurun_out/ak_multi.log
