export SPD_WATCHDOG=500
timeout 300 python scripts/prof_kernels.py inverse 5 > gpurun_out/rb_inv.log 2>&1
SPDKFAC_NO_LOOKAHEAD=1 timeout 300 python scripts/prof_kernels.py inverse 5 > gpurun_out/rb_inv_nola.log 2>&1
timeout 300 python scripts/prof_kernels.py inverse_single 3 > gpurun_out/rb_inv1.log 2>&1
timeout 600 python bench.py --trace gpurun_out/rb_trace.json --timeline --no-cpu-baseline --no-e2e --steps 5 > gpurun_out/rb_bench.log 2>&1; echo "rc=$?" >> gpurun_out/rb_bench.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/rb_launches.csv python bench.py --profile --mode eager --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/rb_ncu_list.log 2>&1; echo "rc=$?" >> gpurun_out/rb_ncu_list.log
