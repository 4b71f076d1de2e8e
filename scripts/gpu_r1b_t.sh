timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:tc3_gemm_kernel<\(spd::Kind\)2, \(int\)3, \(bool\)1" -s 7 -c 1 -o /tmp/rt_upd python scripts/prof_kernels.py inverse 1 > gpurun_out/rt_ncu_upd.log 2>&1; echo "rc=$?" >> gpurun_out/rt_ncu_upd.log
ncu -i /tmp/rt_upd.ncu-rep --page raw --csv > gpurun_out/rt_upd_raw.csv 2>&1
ncu -i /tmp/rt_upd.ncu-rep --page details --csv > gpurun_out/rt_upd_details.csv 2>&1
ncu -i /tmp/rt_upd.ncu-rep --page source --csv --print-source sass > gpurun_out/rt_upd_source.csv 2>&1
