export SPD_WATCHDOG=250
timeout 600 python -m pytest tests/test_gpu_multi.py -q -x > gpurun_out/ad_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/ad_tests.log
for n in 2 4; do
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2954$n bench.py --gpus $n --steps 20 --warmup 3 --no-e2e --timeline > gpurun_out/ad_n$n.log 2>&1; echo "rc=$?" >> gpurun_out/ad_n$n.log
python -c "
import json
for l in open('gpurun_out/ad_n$n.log'):
    if l.startswith('{'):
        d=json.loads(l); print('n$n', d['value'], d['placement_imbalance'], d['timeline_ms'])
        print({k: v['ms_per_step'] for k, v in d['kernel_breakdown'].items() if isinstance(v, dict) and v['ms_per_step']})
" >> gpurun_out/ad_sum.log
done
