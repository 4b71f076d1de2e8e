#!/bin/bash
# Kernel evidence for the fp16-plane inverse (one B200): ncu --set full of the trailing update
# (tc3_gemm_kernel<F16, C-tile>) and the panel GEMM of the batched ResNet-50 inverse, then DRAM bytes
# + duration of every library kernel of one eager bench step.  Each ncu command follows a plain run
# of the same command that exited 0.
export PYTHONPATH=. SPD_WATCHDOG=0
mkdir -p gpurun_out
NCU="ncu --clock-control none --kernel-name-base demangled"
python scripts/prof_drivers.py inverse > gpurun_out/p_inv_plain.log 2>&1 && \
  $NCU --set full --import-source on -k "regex:Kind.0, .int.3, .bool.1" -s 40 -c 3 -o gpurun_out/r2_update_f16 python scripts/prof_drivers.py inverse > gpurun_out/p_upd.log 2>&1
echo "update rc=$?"
$NCU --set full --import-source on -k "regex:Kind.0, .int.3, .bool.0" -s 20 -c 2 -o gpurun_out/r2_panel_f16 python scripts/prof_drivers.py inverse > gpurun_out/p_pan.log 2>&1
echo "panel rc=$?"
ls -la gpurun_out/*.ncu-rep
