#!/bin/bash
# reference arm (CPU, full steps within the wall budget) and the default GPU arm, as the driver runs them
export PYTHONPATH=. SPD_WATCHDOG=900
timeout 900 python bench.py --impl reference --steps 20 --warmup 3 > gpurun_out/r2_ref.json 2> gpurun_out/r2_ref.err
echo "ref rc=$?"; python -c "import json;d=json.loads(open('gpurun_out/r2_ref.json').read().strip().splitlines()[-1]);print(d['value'], d['steps_timed'], d['wall_s'])"
timeout 900 python bench.py --steps 20 --warmup 3 > gpurun_out/r2_gpu_k20.json 2> gpurun_out/r2_gpu_k20.err
echo "gpu rc=$?"; python -c "import json;d=json.loads(open('gpurun_out/r2_gpu_k20.json').read().strip().splitlines()[-1]);print(d['value'], d['e2e']['value'], d['clocks'])"
