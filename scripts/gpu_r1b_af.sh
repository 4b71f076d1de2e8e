timeout 900 python -m pytest tests/test_gpu_multi.py -x -q > gpurun_out/raf_multi.log 2>&1; echo "rc=$?" >> gpurun_out/raf_multi.log
run() { name=$1; n=$2; port=$3; shift 3; timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $port bench.py --gpus $n --steps 10 --warmup 3 "$@" > gpurun_out/raf_$name.log 2>&1; python -c "
import json
for l in open('gpurun_out/raf_$name.log'):
    if l.startswith('{'):
        d=json.loads(l); print('$name', d['value'], d['e2e']['value'] if d.get('e2e') else None, d.get('impl'))
" >> gpurun_out/raf_sum.log; }
run n2 2 29971
run n4 4 29972
run n4ref 4 29973 --impl reference --steps 2 --warmup 1
