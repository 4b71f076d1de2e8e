export SPD_WATCHDOG=250
for i in 1 2; do
for f in 0.85 0.95 0.99; do
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 2957$i bench.py --gpus 2 --steps 20 --warmup 3 --no-e2e --no-cpu-baseline --g1-fraction $f > gpurun_out/ai.log 2>&1
python -c "
import json
for l in open('gpurun_out/ai.log'):
    if l.startswith('{'):
        d=json.loads(l); print('n2 f=$f', d['value'])
" >> gpurun_out/ai_sum.log
done
done
for f in 0.85 0.99; do
timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline --g1-fraction $f > gpurun_out/ai.log 2>&1
python -c "
import json
for l in open('gpurun_out/ai.log'):
    if l.startswith('{'):
        d=json.loads(l); print('n1 f=$f', d['value'])
" >> gpurun_out/ai_sum.log
done
