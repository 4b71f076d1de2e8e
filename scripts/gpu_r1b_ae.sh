export SPD_WATCHDOG=300
timeout 300 python -m pytest tests/test_gpu_linalg.py -x -q -k "inverse" > gpurun_out/rae_pytest_inv.log 2>&1; echo "rc=$?" >> gpurun_out/rae_pytest_inv.log
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/rae_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/rae_pytest.log
timeout 300 python scripts/prof_kernels.py inverse 5 > gpurun_out/rae_inv.log 2>&1
timeout 300 python scripts/prof_kernels.py inverse_single 3 > gpurun_out/rae_inv1.log 2>&1
for i in 1 2; do timeout 300 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/rae_bench_$i.log 2>&1; done
