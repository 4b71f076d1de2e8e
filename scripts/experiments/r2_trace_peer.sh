#!/bin/bash
export PYTHONPATH=. SPD_WATCHDOG=900
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29655"
timeout 900 $TR bench.py --gpus 2 --steps 20 --warmup 5 --no-e2e --trace gpurun_out/r2_trace_peer_n2 > gpurun_out/r2_trace_peer_n2.json 2> gpurun_out/r2_trace_peer_n2.err
echo "rc=$?"; ls gpurun_out/r2_trace_peer_n2*; cat gpurun_out/r2_trace_peer_n2_breakdown.csv 2>/dev/null
python -c "import json;d=json.loads(open('gpurun_out/r2_trace_peer_n2.json').read().strip().splitlines()[-1]);print(d['value'])"
