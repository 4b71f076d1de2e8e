export SPD_WATCHDOG=200
timeout 600 python -m pytest tests/test_gpu_multi.py -q -x > gpurun_out/rr_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/rr_tests.log
for i in 1 2 3; do
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 2953$i bench.py --gpus 2 --steps 10 --warmup 3 --timeline > gpurun_out/rr_n2_$i.log 2>&1; echo "rc=$?" >> gpurun_out/rr_n2_$i.log
python -c "
import json
for l in open('gpurun_out/rr_n2_$i.log'):
    if l.startswith('{'):
        d=json.loads(l); print('run $i', d['value'], d['e2e']['value'], d['timeline_ms'])
" >> gpurun_out/rr_sum.log
tail -1 gpurun_out/rr_n2_$i.log >> gpurun_out/rr_sum.log
done
