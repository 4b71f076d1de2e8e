#!/bin/bash
export PYTHONPATH=. SPD_WATCHDOG=900
timeout 600 python bench.py --steps 20 --warmup 5 --trace gpurun_out/r2_trace > gpurun_out/r2_trace.json 2>gpurun_out/r2_trace.err
echo "trace rc=$?"; cat gpurun_out/r2_trace_breakdown.csv
