export SPD_WATCHDOG=120
timeout 180 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/rc_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/rc_smoke.log
timeout 900 python -m pytest tests/ -q -m gpu -x > gpurun_out/rc_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/rc_tests.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/rc_bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/rc_bench.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --optimizer sgd > gpurun_out/rc_sgd.log 2>&1; echo "sgd rc=$?" >> gpurun_out/rc_sgd.log
