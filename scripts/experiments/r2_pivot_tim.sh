#!/bin/bash
export PYTHONPATH=.
SPDKFAC_LIB=paper_2107_06533_b200/lib/libspdkfac_timing.so timeout 300 python scripts/prof_pivot.py 1024 > gpurun_out/r2_pivot_phases.log 2>&1
echo "phases rc=$?"; grep "b8 sweep" gpurun_out/r2_pivot_phases.log | tail -3
