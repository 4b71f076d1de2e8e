export SPD_WATCHDOG=500
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/rd_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/rd_pytest.log
timeout 600 python bench.py --no-cpu-baseline --trace gpurun_out/rd_trace.json > gpurun_out/rd_bench.log 2>&1; echo "rc=$?" >> gpurun_out/rd_bench.log
timeout 300 python scripts/prof_kernels.py inverse 5 > gpurun_out/rd_inv.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:pivot_kernel -s 4 -c 1 -o /tmp/rd_pivot python scripts/prof_kernels.py inverse 1 > gpurun_out/rd_ncu_pivot.log 2>&1; echo "rc=$?" >> gpurun_out/rd_ncu_pivot.log
ncu -i /tmp/rd_pivot.ncu-rep --page source --csv > gpurun_out/rd_pivot_source.csv 2>&1
ncu -i /tmp/rd_pivot.ncu-rep --page raw --csv > gpurun_out/rd_pivot_raw.csv 2>&1
timeout 1200 ncu --set full --clock-control none --kernel-name-base demangled -k "regex:tc3_gemm_kernel<(\(spd::Kind\))?1|tc3_pair" -s 114 -c 57 -o /tmp/rd_syrk python bench.py --profile --mode eager --steps 1 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/rd_ncu_syrk.log 2>&1; echo "rc=$?" >> gpurun_out/rd_ncu_syrk.log
ncu -i /tmp/rd_syrk.ncu-rep --page raw --csv > gpurun_out/rd_syrk_raw.csv 2>&1
ls -la gpurun_out; du -sh gpurun_out
