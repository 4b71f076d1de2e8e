export SPD_WATCHDOG=200
run() { name=$1; n=$2; port=$3; shift 3; env "$@" timeout 240 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $port bench.py --gpus $n --steps 10 --warmup 3 --no-e2e > gpurun_out/rac_$name.log 2>&1; python -c "
import json
for l in open('gpurun_out/rac_$name.log'):
    if l.startswith('{'):
        d=json.loads(l); print('$name', d['value'])
" >> gpurun_out/rac_sum.log; }
run n2_b9 2 29961 SPDKFAC_GRAD_BUCKET=0.9
run n2_b7 2 29962 SPDKFAC_GRAD_BUCKET=0.7
run n2_b5 2 29963 SPDKFAC_GRAD_BUCKET=0.5
run n2_b97 2 29964 SPDKFAC_GRAD_BUCKET=0.97
run n4_b9 4 29965 SPDKFAC_GRAD_BUCKET=0.9
run n4_b7 4 29966 SPDKFAC_GRAD_BUCKET=0.7
run n4_b5 4 29967 SPDKFAC_GRAD_BUCKET=0.5
run n4_b97 4 29968 SPDKFAC_GRAD_BUCKET=0.97
