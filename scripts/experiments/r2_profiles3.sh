#!/bin/bash
# ncu --set full of the first 16 trailing-update launches (U1/U2 of steps 0-7, incl. the fused bulk
# updates of steps 3 and 7) of the batched ResNet-50 inverse on fp16 planes
export PYTHONPATH=. SPD_WATCHDOG=0
NCU="ncu --clock-control none --kernel-name-base demangled"
python scripts/prof_drivers.py inverse > gpurun_out/p_inv_plain.log 2>&1 && \
  $NCU --set full --import-source on -k "regex:Kind.0, .int.3, .bool.1" -c 16 -o gpurun_out/r2_update_f16b python scripts/prof_drivers.py inverse > gpurun_out/p_upd.log 2>&1
echo "update rc=$?"
