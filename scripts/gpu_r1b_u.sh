export SPD_WATCHDOG=200
run() { name=$1; n=$2; port=$3; shift 3; timeout 240 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $port bench.py --gpus $n --steps 10 --warmup 3 --no-e2e "$@" > gpurun_out/ru_$name.log 2>&1; python -c "
import json
for l in open('gpurun_out/ru_$name.log'):
    if l.startswith('{'):
        d=json.loads(l); print('$name', d['value'], d['config']['scheme'], d['config']['fusion'], d['config']['placement'], d.get('placement_imbalance'))
" >> gpurun_out/ru_sum.log; }
run n4_spd 4 29901 --scheme spdkfac
run n4_mpd 4 29902 --scheme mpdkfac
run n4_d 4 29903 --scheme dkfac
run n4_nopipe 4 29904 --scheme -pipe+lbp
run n4_nolbp 4 29905 --scheme +pipe-lbp
run n2_spd 2 29906 --scheme spdkfac
run n2_mpd 2 29907 --scheme mpdkfac
run n2_d 2 29908 --scheme dkfac
run n4_spd_b 4 29909 --scheme spdkfac
