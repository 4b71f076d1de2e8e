SPDKFAC_NO_LOOKAHEAD=1 timeout 300 python scripts/prof_kernels.py inverse_single 3 > gpurun_out/pc_nola.log 2>&1
timeout 300 python scripts/prof_kernels.py inverse_single 1 > gpurun_out/pc_plain.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"pivot_kernel" -s 5 -c 1 -o gpurun_out/prof_pivot2 python scripts/prof_kernels.py inverse_single 1 > gpurun_out/pc_ncu.log 2>&1
echo "rc=$?" >> gpurun_out/pc_ncu.log
