export SPD_WATCHDOG=250
timeout 600 python -m pytest tests/test_gpu_multi.py -q -x > gpurun_out/ae_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/ae_tests.log
for i in 1 2 3; do
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 2955$i bench.py --gpus 2 --steps 20 --warmup 3 --no-e2e --no-cpu-baseline --timeline > gpurun_out/ae_n2.log 2>&1; echo "rc=$?" >> gpurun_out/ae_sum.log
python -c "
import json
for l in open('gpurun_out/ae_n2.log'):
    if l.startswith('{'):
        d=json.loads(l); print('n2', d['value'], d['timeline_ms'])
" >> gpurun_out/ae_sum.log
done
