export SPD_WATCHDOG=300
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/rz_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/rz_pytest.log
for i in 1 2 3; do timeout 300 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/rz_bench_$i.log 2>&1; done
