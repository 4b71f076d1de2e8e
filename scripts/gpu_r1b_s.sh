export SPD_WATCHDOG=300
timeout 300 python -m pytest tests/test_gpu_linalg.py -x -q > gpurun_out/rs_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/rs_pytest.log
timeout 300 python scripts/prof_kernels.py inverse 5 > gpurun_out/rs_inv.log 2>&1
for i in 1 2 3; do timeout 300 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/rs_bench_$i.log 2>&1; done
