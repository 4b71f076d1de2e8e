export SPD_WATCHDOG=200
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q > gpurun_out/raa_multi.log 2>&1; echo "rc=$?" >> gpurun_out/raa_multi.log
run() { name=$1; n=$2; port=$3; shift 3; timeout 240 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $port bench.py --gpus $n --steps 10 --warmup 3 "$@" > gpurun_out/raa_$name.log 2>&1; python -c "
import json
for l in open('gpurun_out/raa_$name.log'):
    if l.startswith('{'):
        d=json.loads(l); print('$name', d['value'], d['e2e']['value'] if d.get('e2e') else None)
" >> gpurun_out/raa_sum.log; }
run n2 2 29951
run n4 4 29952
run n2_trace 2 29953 --trace gpurun_out/raa_trace_n2.json --no-e2e
run n4b 4 29954
run n2b 2 29955
