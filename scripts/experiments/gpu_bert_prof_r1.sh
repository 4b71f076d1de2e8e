#!/bin/bash
# configs[4] launch list (serialised, cold-cache per-kernel times) for the per-category share.
mkdir -p gpurun_out
export SPD_WATCHDOG=0
timeout 700 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/bert_launches.csv python bench.py --model bert_base_linears --profile --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bert_ncu_list.log 2>&1; echo "rc=$?" >> gpurun_out/bert_ncu_list.log
tail -2 gpurun_out/bert_ncu_list.log; wc -l gpurun_out/bert_launches.csv
