export SPD_WATCHDOG=500
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/rc_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/rc_pytest.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/rc_bench.log 2>&1; echo "rc=$?" >> gpurun_out/rc_bench.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:pivot_kernel -s 4 -c 2 -o gpurun_out/rc_pivot python scripts/prof_kernels.py inverse 1 > gpurun_out/rc_ncu_pivot.log 2>&1; echo "rc=$?" >> gpurun_out/rc_ncu_pivot.log
timeout 1200 ncu --set full --clock-control none --kernel-name-base demangled -k "regex:tc3_gemm_kernel<(\(spd::Kind\))?1|tc3_pair" -s 114 -c 57 -o gpurun_out/rc_syrk_step python bench.py --profile --mode eager --steps 1 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/rc_ncu_syrk.log 2>&1; echo "rc=$?" >> gpurun_out/rc_ncu_syrk.log
