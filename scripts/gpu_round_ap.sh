export SPD_WATCHDOG=250
run() {
  env $1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $3 --master-addr 127.0.0.1 --master-port $2 bench.py --gpus $3 --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ap.log 2>&1
  python -c "
import json
for l in open('gpurun_out/ap.log'):
    if l.startswith('{'):
        d=json.loads(l); print('n$3 $1', d['value'])
" >> gpurun_out/ap_sum.log
}
NCCL_DEBUG=INFO timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29650 bench.py --gpus 4 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ap_debug.log 2>&1
for n in 4 2; do
run "X=1" 2966$n $n
run "NCCL_MIN_NCHANNELS=32" 2967$n $n
run "NCCL_PROTO=Simple" 2968$n $n
run "NCCL_ALGO=Ring" 2969$n $n
run "NCCL_NVLS_ENABLE=0" 2970$n $n
done
