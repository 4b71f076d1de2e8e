#!/bin/bash
# ncu launch list (serialised kernel durations) of the batched ResNet-50 inverse, pairs on / off.
export PYTHONPATH=. SPD_WATCHDOG=0
for pr in 1 0; do
  SPDKFAC_UPDATE_PAIRS=$pr python scripts/prof_drivers.py inverse > /dev/null 2>&1 && \
  SPDKFAC_UPDATE_PAIRS=$pr ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:tc3 --csv python scripts/prof_drivers.py inverse > gpurun_out/pairs_ncu$pr.csv 2>/dev/null
  echo "pairs=$pr rc=$?"
done
