timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:tc3_gemm_kernel<\(spd::Kind\)2, \(int\)2" -s 2 -c 4 -o /tmp/rj_upd python scripts/prof_kernels.py inverse 1 > gpurun_out/rj_ncu_upd.log 2>&1; echo "rc=$?" >> gpurun_out/rj_ncu_upd.log
ncu -i /tmp/rj_upd.ncu-rep --page raw --csv > gpurun_out/rj_upd_raw.csv 2>&1
ncu -i /tmp/rj_upd.ncu-rep --page details --csv > gpurun_out/rj_upd_details.csv 2>&1
timeout 600 ncu --set full --clock-control none --kernel-name-base demangled -k "regex:stage_rows|stage_im2col|stage_spatial" -s 20 -c 12 -o /tmp/rj_stage python bench.py --profile --mode eager --steps 1 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/rj_ncu_stage.log 2>&1; echo "rc=$?" >> gpurun_out/rj_ncu_stage.log
ncu -i /tmp/rj_stage.ncu-rep --page raw --csv > gpurun_out/rj_stage_raw.csv 2>&1
