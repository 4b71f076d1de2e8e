export SPD_WATCHDOG=600
timeout 600 python bench.py --model resnet50 --batch 32 --steps 10 --warmup 3 --no-cpu-baseline --optimizer sgd > gpurun_out/rah_r50_sgd.log 2>&1; echo "rc=$?" >> gpurun_out/rah_r50_sgd.log
timeout 600 python bench.py --model densenet201 --batch 16 --steps 5 --warmup 3 --no-cpu-baseline --optimizer sgd > gpurun_out/rah_densenet_sgd.log 2>&1; echo "rc=$?" >> gpurun_out/rah_densenet_sgd.log
timeout 600 python bench.py --model resnet152 --batch 32 --steps 5 --warmup 3 --no-cpu-baseline --optimizer sgd > gpurun_out/rah_r152_sgd.log 2>&1; echo "rc=$?" >> gpurun_out/rah_r152_sgd.log
