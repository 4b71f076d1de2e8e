export SPD_WATCHDOG=250
timeout 600 python -m pytest tests/test_gpu_multi.py -q -x > gpurun_out/rs_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/rs_tests.log
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29541 bench.py --gpus 4 --steps 10 --warmup 3 --timeline > gpurun_out/rs_n4.log 2>&1; echo "rc=$?" >> gpurun_out/rs_n4.log
python -c "
import json
for l in open('gpurun_out/rs_n4.log'):
    if l.startswith('{'):
        d=json.loads(l); print('n4', d['value'], d['e2e']['value'], d['placement_imbalance'], d['timeline_ms'])
        print({k: v['ms_per_step'] for k, v in d['kernel_breakdown'].items() if isinstance(v, dict) and v['ms_per_step']})
" > gpurun_out/rs_sum.log
