export SPD_WATCHDOG=250
run() {
  env $1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $3 --master-addr 127.0.0.1 --master-port $2 bench.py --gpus $3 --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/as.log 2>&1
  python -c "
import json
for l in open('gpurun_out/as.log'):
    if l.startswith('{'):
        d=json.loads(l); print('n$3 $1', d['value'])
" >> gpurun_out/as_sum.log
}
NCCL_DEBUG=INFO NCCL_DEBUG_SUBSYS=TUNING timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29850 bench.py --gpus 4 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/as_debug.log 2>&1
run "X=1" 29851 4
run "NCCL_PROTO=LL128" 29852 4
run "NCCL_ALGO=NVLS" 29853 4
run "NCCL_PROTO=LL128,Simple" 29854 4
run "NCCL_ALGO=NVLS,Ring" 29855 4
run "NCCL_PROTO=LL128" 29856 2
