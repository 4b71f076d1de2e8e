export SPD_WATCHDOG=500
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/rg_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/rg_pytest.log
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:tc3_gemm_kernel<(\(spd::Kind\))?2, 2" -s 2 -c 6 -o /tmp/rg_upd python scripts/prof_kernels.py inverse 1 > gpurun_out/rg_ncu_upd.log 2>&1; echo "rc=$?" >> gpurun_out/rg_ncu_upd.log
ncu -i /tmp/rg_upd.ncu-rep --page raw --csv > gpurun_out/rg_upd_raw.csv 2>&1
ncu -i /tmp/rg_upd.ncu-rep --page details --csv > gpurun_out/rg_upd_details.csv 2>&1
ncu -i /tmp/rg_upd.ncu-rep --page source --csv --print-source sass > gpurun_out/rg_upd_source.csv 2>&1
ls -la gpurun_out | tail -5
