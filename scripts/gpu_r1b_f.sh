export SPD_WATCHDOG=500
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/rf_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/rf_pytest.log
timeout 600 python bench.py --no-cpu-baseline --trace gpurun_out/rf_trace.json > gpurun_out/rf_bench.log 2>&1; echo "rc=$?" >> gpurun_out/rf_bench.log
