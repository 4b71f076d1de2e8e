#!/bin/bash
# Round-2 kernel evidence (one B200): ncu --set full of the inverse trailing update, the pivot
# sweep and the factor staging kernels (isolated drivers), then DRAM bytes + duration of every
# library kernel of one eager bench step (the per-category traffic behind roofline.traffic).
# Each ncu command follows a plain run of the same command that exited 0.
export PYTHONPATH=. SPD_WATCHDOG=0
mkdir -p gpurun_out
NCU="ncu --clock-control none --kernel-name-base demangled"
python scripts/prof_drivers.py inverse > gpurun_out/p_inv_plain.log 2>&1 && \
  $NCU --set full --import-source on -k "regex:3, true" -s 40 -c 3 -o gpurun_out/r2_update python scripts/prof_drivers.py inverse > gpurun_out/p_upd.log 2>&1
echo "update rc=$?"
$NCU --set full --import-source on -k "regex:pivot_kernel" -s 36 -c 2 -o gpurun_out/r2_pivot python scripts/prof_drivers.py inverse > gpurun_out/p_piv.log 2>&1
echo "pivot rc=$?"
python scripts/prof_drivers.py stage > gpurun_out/p_stage_plain.log 2>&1 && \
  $NCU --set full --import-source on -k "regex:stage_" -c 3 -o gpurun_out/r2_stage python scripts/prof_drivers.py stage > gpurun_out/p_stage.log 2>&1
echo "stage rc=$?"
python bench.py --profile --mode eager --steps 2 --warmup 3 > gpurun_out/p_bench_plain.log 2>&1 && \
  $NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --profile-from-start off --csv \
  --log-file gpurun_out/r2_step_traffic.csv python bench.py --profile --mode eager --steps 2 --warmup 3 --ncu-range > gpurun_out/p_bench_ncu.log 2>&1
echo "step rc=$?"
