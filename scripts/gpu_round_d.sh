export SPD_WATCHDOG=120
timeout 600 python -m pytest tests/test_gpu_linalg.py -q -x -k "inverse" > gpurun_out/rd_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/rd_tests.log
timeout 300 python scripts/prof_kernels.py inverse 3 > gpurun_out/rd_prof.log 2>&1
