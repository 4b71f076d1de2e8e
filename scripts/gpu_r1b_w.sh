export SPD_WATCHDOG=200
run() { name=$1; n=$2; port=$3; shift 3; env "$@" timeout 240 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $port bench.py --gpus $n --steps 10 --warmup 3 --no-e2e > gpurun_out/rw_$name.log 2>&1; python -c "
import json
for l in open('gpurun_out/rw_$name.log'):
    if l.startswith('{'):
        d=json.loads(l); print('$name', d['value'])
" >> gpurun_out/rw_sum.log; }
run n2_a2 2 29931 SPDKFAC_A_BCAST_AFTER=2
run n2_a1 2 29932 SPDKFAC_A_BCAST_AFTER=1
run n2_a0 2 29933 SPDKFAC_A_BCAST_AFTER=0
run n4_a2 4 29934 SPDKFAC_A_BCAST_AFTER=2
run n4_a1 4 29935 SPDKFAC_A_BCAST_AFTER=1
run n4_a0 4 29936 SPDKFAC_A_BCAST_AFTER=0
run n2_a2b 2 29937 SPDKFAC_A_BCAST_AFTER=2
run n2_a1b 2 29938 SPDKFAC_A_BCAST_AFTER=1
