#!/bin/bash
# Inverse-update item order A/B (isolated batched ResNet-50 inverse + the bench), then one ncu --set
# full capture of the update kernel (matrix-major order, the default).
export PYTHONPATH=. SPD_WATCHDOG=0
for o in matrix nk; do
  SPDKFAC_UPDATE_ORDER=$o timeout 300 python scripts/bench_inverse.py > gpurun_out/inv_$o.json 2>&1
  python -c "import json;d=json.load(open('gpurun_out/inv_$o.json'));print('$o', {k:(d[k]['ms_total'], d[k]['cats'].get('inv_update',{}).get('ms')) for k in ('d4608','resnet50_all108')})"
  SPDKFAC_UPDATE_ORDER=$o timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/ab_upd_$o.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/ab_upd_$o.json').read().strip().splitlines()[-1]);print('$o bench', d['value'], {k:(v['kernel_ms_per_step'], v['frac']) for k,v in d['roofline_kernels'].items()})"
done
python scripts/prof_drivers.py inverse > /dev/null 2>&1 && ncu --clock-control none --kernel-name-base demangled --set full --import-source on -k "regex:3, true" -s 40 -c 3 -o gpurun_out/r2_update python scripts/prof_drivers.py inverse > gpurun_out/p_upd.log 2>&1
echo "ncu rc=$?"; tail -2 gpurun_out/p_upd.log
