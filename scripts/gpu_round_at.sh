export SPD_WATCHDOG=250
timeout 600 python -m pytest tests/test_gpu_multi.py -q -x > gpurun_out/at_multi.log 2>&1; echo "rc=$?" >> gpurun_out/at_multi.log
for i in 1 2; do
for n in 2 4; do
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29700 + n*10 + i)) bench.py --gpus $n --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/at.log 2>&1
python -c "
import json
for l in open('gpurun_out/at.log'):
    if l.startswith('{'):
        d=json.loads(l); print('n$n', d['value'])
" >> gpurun_out/at_sum.log
done
done
