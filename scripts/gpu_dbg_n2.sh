export SPD_WATCHDOG=150
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29534 bench.py --gpus 2 --steps 4 --warmup 3 > gpurun_out/dbg_graph2.log 2>&1; echo "graph+e2e rc=$?" >> gpurun_out/dbg_graph2.log
