export SPD_WATCHDOG=500
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/rq_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/rq_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/rq_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/rq_smoke.log
timeout 600 python bench.py > gpurun_out/rq_bench.log 2>&1; echo "rc=$?" >> gpurun_out/rq_bench.log
timeout 600 python bench.py --no-cpu-baseline --no-e2e --trace gpurun_out/rq_trace.json > gpurun_out/rq_bench_trace.log 2>&1; echo "rc=$?" >> gpurun_out/rq_bench_trace.log
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/rq_ref.log 2>&1; echo "rc=$?" >> gpurun_out/rq_ref.log
unset SPD_WATCHDOG
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/rq_launches.csv python bench.py --profile --mode eager --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/rq_ncu_list.log 2>&1; echo "rc=$?" >> gpurun_out/rq_ncu_list.log
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:tc3_gemm_kernel<\(spd::Kind\)2, \(int\)3, \(bool\)1" -s 2 -c 3 -o /tmp/rq_upd python scripts/prof_kernels.py inverse 1 > gpurun_out/rq_ncu_upd.log 2>&1; echo "rc=$?" >> gpurun_out/rq_ncu_upd.log
ncu -i /tmp/rq_upd.ncu-rep --page raw --csv > gpurun_out/rq_upd_raw.csv 2>&1
