export SPD_WATCHDOG=120
timeout 900 python -m pytest tests/test_gpu_linalg.py tests/test_gpu_optimizer.py -q -x > gpurun_out/rp_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/rp_tests.log
timeout 300 python scripts/prof_kernels.py inverse_single 3 > gpurun_out/rp_a.log 2>&1
timeout 300 python scripts/prof_kernels.py inverse 3 > gpurun_out/rp_b.log 2>&1
