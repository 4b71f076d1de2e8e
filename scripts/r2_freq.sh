#!/bin/bash
# Update frequencies in graph mode (simulator.py:126,377): amortised iteration ms at inv_update_freq
# 1 / 10 and factor decay 0 / 0.95 (20 timed steps = 2 inversion periods); then the ncu capture of the
# inverse update kernel and the reference arm (every layer per step).
export PYTHONPATH=. SPD_WATCHDOG=900
for cfg in "1 0.0" "10 0.0" "1 0.95" "10 0.95"; do
  set -- $cfg
  timeout 900 python bench.py --steps 20 --warmup 5 --inv-freq $1 --factor-decay $2 --no-cpu-baseline > gpurun_out/r2_freq_i$1_r$2.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/r2_freq_i$1_r$2.json').read().strip().splitlines()[-1]);print('inv_freq $1 decay $2', d['value'], d['e2e']['value'], d['per_step_ms'][:12])"
done
python scripts/prof_drivers.py inverse > /dev/null 2>&1 && ncu --clock-control none --set full --import-source on -k "regex:tc3_gemm_kernel<2, 3, 1" -s 40 -c 3 -o gpurun_out/r2_update python scripts/prof_drivers.py inverse > gpurun_out/p_upd.log 2>&1
echo "ncu rc=$?"; ls gpurun_out | grep r2_update
timeout 1500 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/r2_final_ref.json 2> gpurun_out/r2_final_ref.err
echo "ref rc=$?"; python -c "import json;d=json.loads(open('gpurun_out/r2_final_ref.json').read().strip().splitlines()[-1]);print('ref', d['value'], d['wall_s'], d['per_step_ms'][:5])"
