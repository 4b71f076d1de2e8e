timeout 300 python scripts/prof_kernels.py inverse_single 3 > gpurun_out/ro_a.log 2>&1
SPDKFAC_NO_LOOKAHEAD=1 timeout 300 python scripts/prof_kernels.py inverse_single 3 > gpurun_out/ro_b.log 2>&1
SPDKFAC_NO_LOOKAHEAD=1 timeout 300 python scripts/prof_kernels.py inverse 3 > gpurun_out/ro_c.log 2>&1
