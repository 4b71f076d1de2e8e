export SPD_WATCHDOG=500
timeout 600 python bench.py --no-cpu-baseline --trace gpurun_out/re_trace.json > gpurun_out/re_bench.log 2>&1; echo "rc=$?" >> gpurun_out/re_bench.log
timeout 600 python bench.py --no-cpu-baseline --no-e2e --launch-groups fusion > gpurun_out/re_bench_fusion.log 2>&1; echo "rc=$?" >> gpurun_out/re_bench_fusion.log
timeout 600 python -m pytest tests/test_gpu_optimizer.py -x -q > gpurun_out/re_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/re_pytest.log
