export SPD_WATCHDOG=500
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/ra_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/ra_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/ra_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/ra_smoke.log
timeout 600 python bench.py > gpurun_out/ra_bench.log 2>&1; echo "rc=$?" >> gpurun_out/ra_bench.log
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/ra_ref.log 2>&1; echo "rc=$?" >> gpurun_out/ra_ref.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ra_launches.csv python bench.py --profile --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ra_ncu_list.log 2>&1; echo "rc=$?" >> gpurun_out/ra_ncu_list.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tc3 -s 250 -c 12 -o gpurun_out/ra_syrk python bench.py --profile --mode eager --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ra_ncu_syrk.log 2>&1; echo "rc=$?" >> gpurun_out/ra_ncu_syrk.log
