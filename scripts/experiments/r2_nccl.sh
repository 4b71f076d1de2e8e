#!/bin/bash
# NCCL channel count vs compute interference at N (bench with the default params)
N=${1:-2}
export PYTHONPATH=. SPD_WATCHDOG=900
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
run() {  # name, env
  env $2 timeout 900 $TR --master-port $((29620 + RANDOM % 300)) bench.py --gpus $N --steps 20 --warmup 5 --no-e2e > gpurun_out/r2n_$1.json 2> gpurun_out/r2n_$1.err
  python -c "import json;d=json.loads(open('gpurun_out/r2n_$1.json').read().strip().splitlines()[-1]);print('$1', d['value'])" || tail -3 gpurun_out/r2n_$1.err
}
NCCL_DEBUG=INFO timeout 600 $TR --master-port 29601 bench.py --gpus $N --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2> gpurun_out/r2n_debug.err
grep -E "NVLS|Channel|nchannels|algorithm|Using" gpurun_out/r2n_debug.err | head -8
run default ""
run ch4 "NCCL_MAX_NCHANNELS=4"
run ch8 "NCCL_MAX_NCHANNELS=8"
run ch16 "NCCL_MAX_NCHANNELS=16"
run nvls0 "NCCL_NVLS_ENABLE=0"
