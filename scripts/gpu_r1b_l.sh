export SPD_WATCHDOG=500
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/rl_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/rl_pytest.log
timeout 600 python bench.py --trace gpurun_out/rl_trace.json > gpurun_out/rl_bench.log 2>&1; echo "rc=$?" >> gpurun_out/rl_bench.log
unset SPD_WATCHDOG
timeout 1200 ncu --set full --clock-control none --profile-from-start off --kernel-name-base demangled -k "regex:tc3_gemm_kernel<\(spd::Kind\)1|tc3_pair" -o /tmp/rl_syrk python bench.py --profile --mode eager --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --ncu-range > gpurun_out/rl_ncu_syrk.log 2>&1; echo "rc=$?" >> gpurun_out/rl_ncu_syrk.log
ncu -i /tmp/rl_syrk.ncu-rep --page raw --csv > gpurun_out/rl_syrk_raw.csv 2>&1
