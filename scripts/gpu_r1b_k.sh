export SPD_WATCHDOG=500
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/rk_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/rk_pytest.log
timeout 600 python bench.py > gpurun_out/rk_bench.log 2>&1; echo "rc=$?" >> gpurun_out/rk_bench.log
timeout 1200 ncu --set full --clock-control none --kernel-name-base demangled -k "regex:tc3_gemm_kernel<\(spd::Kind\)1|tc3_pair" -c 80 -o /tmp/rk_syrk python bench.py --profile --mode eager --steps 1 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/rk_ncu_syrk.log 2>&1; echo "rc=$?" >> gpurun_out/rk_ncu_syrk.log
ncu -i /tmp/rk_syrk.ncu-rep --page raw --csv > gpurun_out/rk_syrk_raw.csv 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/rk_launches.csv python bench.py --profile --mode eager --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/rk_ncu_list.log 2>&1; echo "rc=$?" >> gpurun_out/rk_ncu_list.log
