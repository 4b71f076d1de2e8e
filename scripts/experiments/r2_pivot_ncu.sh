#!/bin/bash
# ncu --set full of the v3 pivot sweep (one d = 1024 inverse, 8 pivot launches x 2 runs; capture 2)
export PYTHONPATH=.
timeout 300 python scripts/prof_pivot.py 1024 && \
timeout 900 ncu --set full --import-source on --clock-control none -k regex:pivot_kernel -c 2 -o gpurun_out/r2_pivot_v3 -f python scripts/prof_pivot.py 1024 > gpurun_out/r2_pivot_v3_ncu.log 2>&1
echo "ncu rc=$?"; tail -3 gpurun_out/r2_pivot_v3_ncu.log
