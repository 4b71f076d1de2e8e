export SPD_WATCHDOG=250
run() {
  env $1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $2 bench.py --gpus 2 --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ao.log 2>&1
  python -c "
import json
for l in open('gpurun_out/ao.log'):
    if l.startswith('{'):
        d=json.loads(l); print('$1', d['value'])
" >> gpurun_out/ao_sum.log
}
for i in 1 2; do
run "X=1" 2959$i
run "NCCL_MAX_NCHANNELS=8" 2960$i
run "NCCL_MAX_NCHANNELS=4" 2961$i
run "NCCL_NVLS_ENABLE=1" 2962$i
run "NCCL_MAX_NCHANNELS=2" 2963$i
done
