#!/bin/bash
export PYTHONPATH=. SPD_WATCHDOG=900
timeout 600 python bench.py --steps 20 --warmup 5 --no-e2e --trace gpurun_out/r2_trace_n1b > gpurun_out/r2_trace_n1b.json 2> gpurun_out/r2_trace_n1b.err
echo "rc=$?"; cat gpurun_out/r2_trace_n1b_breakdown.csv
