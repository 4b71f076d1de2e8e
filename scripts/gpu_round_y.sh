export SPD_WATCHDOG=250
(cd _ab_old && timeout 300 python scripts/prof_kernels.py stage 5 > ../gpurun_out/y_old.log 2>&1)
timeout 300 python scripts/prof_kernels.py stage 5 > gpurun_out/y_new.log 2>&1
