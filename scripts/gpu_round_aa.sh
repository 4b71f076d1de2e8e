export SPD_WATCHDOG=250
(cd _ab_old && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base mangled --kernel-name regex:3spd --csv --log-file ../gpurun_out/aa_old.csv python bench.py --profile --mode eager --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > ../gpurun_out/aa_old.log 2>&1)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base mangled --kernel-name regex:3spd --csv --log-file gpurun_out/aa_new.csv python bench.py --profile --mode eager --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/aa_new.log 2>&1
