export SPD_WATCHDOG=500
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/rad_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/rad_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/rad_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/rad_smoke.log
unset SPD_WATCHDOG
timeout 600 python bench.py > gpurun_out/rad_bench.log 2>&1; echo "rc=$?" >> gpurun_out/rad_bench.log
