timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/mb_n1.log 2>&1
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --stats-off > gpurun_out/mb_n1_nostats.log 2>&1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 5 --warmup 3 > gpurun_out/mb_n2.log 2>&1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29534 bench.py --gpus 2 --steps 5 --warmup 3 --stats-off > gpurun_out/mb_n2_nostats.log 2>&1
