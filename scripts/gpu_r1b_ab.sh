export SPD_WATCHDOG=500
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/rab_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/rab_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/rab_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/rab_smoke.log
timeout 600 python bench.py > gpurun_out/rab_bench.log 2>&1; echo "rc=$?" >> gpurun_out/rab_bench.log
timeout 600 python bench.py --no-cpu-baseline --no-e2e --trace gpurun_out/rab_trace.json > gpurun_out/rab_bench_trace.log 2>&1; echo "rc=$?" >> gpurun_out/rab_bench_trace.log
unset SPD_WATCHDOG
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/rab_launches.csv python bench.py --profile --mode eager --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/rab_ncu_list.log 2>&1; echo "rc=$?" >> gpurun_out/rab_ncu_list.log
timeout 1200 ncu --set full --clock-control none --profile-from-start off --kernel-name-base demangled -k "regex:tc3_gemm_kernel<\(spd::Kind\)1|tc3_pair" -o /tmp/rab_syrk python bench.py --profile --mode eager --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --ncu-range > gpurun_out/rab_ncu_syrk.log 2>&1; echo "rc=$?" >> gpurun_out/rab_ncu_syrk.log
ncu -i /tmp/rab_syrk.ncu-rep --page raw --csv > gpurun_out/rab_syrk_raw.csv 2>&1
