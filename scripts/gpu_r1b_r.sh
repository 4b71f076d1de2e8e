export SPD_WATCHDOG=200
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q > gpurun_out/rr_multi.log 2>&1; echo "rc=$?" >> gpurun_out/rr_multi.log
run() { name=$1; n=$2; port=$3; shift 3; env "$@" timeout 240 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $port bench.py --gpus $n --steps 10 --warmup 3 $BARGS > gpurun_out/rr_$name.log 2>&1; python -c "
import json
for l in open('gpurun_out/rr_$name.log'):
    if l.startswith('{'):
        d=json.loads(l); print('$name', d['value'], d['e2e']['value'] if d.get('e2e') else None)
" >> gpurun_out/rr_sum.log; }
BARGS="" run n2 2 29801 X=1
BARGS="" run n4 4 29802 X=1
BARGS="" run n2_simple 2 29803 NCCL_PROTO=Simple
BARGS="" run n4_simple 4 29804 NCCL_PROTO=Simple
BARGS="" run n4_ll128 4 29805 NCCL_PROTO=LL128,Simple
BARGS="--trace gpurun_out/rr_trace_n2.json" run n2_trace 2 29806 X=1
BARGS="" run n4b 4 29807 X=1
