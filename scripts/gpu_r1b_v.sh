export SPD_WATCHDOG=200
run() { name=$1; n=$2; port=$3; shift 3; timeout 240 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $port bench.py --gpus $n --steps 10 --warmup 3 --no-e2e "$@" > gpurun_out/rv_$name.log 2>&1; python -c "
import json
for l in open('gpurun_out/rv_$name.log'):
    if l.startswith('{'):
        d=json.loads(l); print('$name', d['value'], d['config']['scheme'], d['config']['fusion'], d['config']['placement'])
" >> gpurun_out/rv_sum.log; }
run n4_nopipe 4 29921 --scheme spdkfac-nopipe
run n2_nopipe 2 29922 --scheme spdkfac-nopipe
run n2_nolbp 2 29923 --scheme spdkfac-nolbp
run n4_nolbp 4 29924 --scheme spdkfac-nolbp
run n4_mpd 4 29925 --scheme mpdkfac
run n4_d 4 29926 --scheme dkfac
