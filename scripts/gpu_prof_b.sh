export SPD_WATCHDOG=120
timeout 900 python -m pytest tests/ -q -m gpu -x > gpurun_out/pb_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/pb_tests.log
# launch list of one bench step (eager, so kernel names are visible per launch)
timeout 600 python bench.py --steps 2 --warmup 1 --profile --mode eager > gpurun_out/pb_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/pb_launches.csv python bench.py --steps 2 --warmup 1 --profile --mode eager > gpurun_out/pb_ncu1.log 2>&1
echo "launches rc=$?" >> gpurun_out/pb_ncu1.log
# full capture of the factor SYRK kernel (layer4 conv2 A, layer1 conv2 A) and the update kernel
timeout 300 python scripts/prof_kernels.py factor 1 > gpurun_out/pb_plain2.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"tc3_gemm_kernel|stage_" -c 6 -o gpurun_out/prof_factor python scripts/prof_kernels.py factor 1 > gpurun_out/pb_ncu2.log 2>&1
echo "factor prof rc=$?" >> gpurun_out/pb_ncu2.log
