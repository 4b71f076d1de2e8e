#!/bin/bash
# refreshed kernel evidence: ncu --set full of the pivot sweep (v3, FFMA2) and of the first 12
# trailing-update launches (fp16 planes, kFuse 8 schedule) of the batched ResNet-50 inverse; launch
# list + DRAM bytes of one eager bench step
export PYTHONPATH=. SPD_WATCHDOG=0
NCU="ncu --clock-control none --kernel-name-base demangled"
python scripts/prof_drivers.py inverse > gpurun_out/p_inv_plain.log 2>&1 && \
  $NCU --set full --import-source on -k "regex:pivot_kernel" -s 36 -c 2 -o gpurun_out/r2_pivot_ffma2 python scripts/prof_drivers.py inverse > gpurun_out/p_piv.log 2>&1
echo "pivot rc=$?"
$NCU --set full --import-source on -k "regex:Kind.0, .int.3, .bool.1" -c 12 -o gpurun_out/r2_update_f16c python scripts/prof_drivers.py inverse > gpurun_out/p_upd.log 2>&1
echo "update rc=$?"
python bench.py --profile --mode eager --steps 2 --warmup 3 > gpurun_out/p_bench_plain.log 2>&1 && \
  $NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --profile-from-start off --csv \
  --log-file gpurun_out/r2_step_traffic.csv python bench.py --profile --mode eager --steps 2 --warmup 3 --ncu-range > gpurun_out/p_bench_ncu.log 2>&1
echo "step rc=$?"
