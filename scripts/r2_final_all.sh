#!/bin/bash
# full single-GPU suite + smoke + default bench, then the multi-rank tests and an N=2 bench (run with --gpus 2)
export PYTHONPATH=. SPD_WATCHDOG=900
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2fa_tests.log 2>&1
echo "tests rc=$?"; tail -1 gpurun_out/r2fa_tests.log; grep -E "FAILED" gpurun_out/r2fa_tests.log | head
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2fa_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/r2fa_smoke.log
CUDA_VISIBLE_DEVICES=0 timeout 900 python bench.py > gpurun_out/r2fa_bench.json 2> gpurun_out/r2fa_bench.err
echo "bench rc=$?"; python -c "import json;d=json.loads(open('gpurun_out/r2fa_bench.json').read().strip().splitlines()[-1]);print('n1', d['value'], d['e2e']['value'], d['clocks']['reasons'])"
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29677"
timeout 600 $TR bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/r2fa_bench_n2.json 2> gpurun_out/r2fa_bench_n2.err
python -c "import json;d=json.loads(open('gpurun_out/r2fa_bench_n2.json').read().strip().splitlines()[-1]);print('n2', d['value'], d['e2e']['value'])"
