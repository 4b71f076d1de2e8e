timeout 300 python scripts/prof_kernels.py all 3 > gpurun_out/pa_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"pivot_kernel|tc3_gemm_kernel" -s 40 -c 3 -o gpurun_out/prof_inv python scripts/prof_kernels.py inverse 1 > gpurun_out/pa_ncu.log 2>&1
echo "rc=$?" >> gpurun_out/pa_ncu.log
