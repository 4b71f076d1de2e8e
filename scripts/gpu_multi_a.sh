export SPD_WATCHDOG=120
timeout 900 python -m pytest tests/test_gpu_multi.py -q -x -k two_rank > gpurun_out/ma_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/ma_tests.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 5 --warmup 3 > gpurun_out/ma_bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/ma_bench.log
