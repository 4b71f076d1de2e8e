export SPD_WATCHDOG=120
timeout 180 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/rq_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/rq_smoke.log
timeout 900 python -m pytest tests/ -q -m gpu -x > gpurun_out/rq_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/rq_tests.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --timeline > gpurun_out/rq_n1.log 2>&1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 10 --warmup 3 --timeline > gpurun_out/rq_n2.log 2>&1
for f in rq_n1 rq_n2; do python -c "
import json
for l in open('gpurun_out/$f.log'):
    if l.startswith('{'):
        d=json.loads(l); print('$f', d['value'], d['e2e']['value'], d['roofline']['achieved'], d['gpu_launches'], d['timeline_ms'])
        print({k: v['ms_per_step'] for k, v in d['kernel_breakdown'].items() if isinstance(v, dict) and v['ms_per_step']})
" >> gpurun_out/rq_sum.log; done
