export SPD_WATCHDOG=600
timeout 600 python bench.py --model densenet201 --batch 16 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/rag_densenet.log 2>&1; echo "rc=$?" >> gpurun_out/rag_densenet.log
timeout 600 python bench.py --model resnet152 --batch 32 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/rag_r152.log 2>&1; echo "rc=$?" >> gpurun_out/rag_r152.log
timeout 600 python bench.py --model densenet201 --batch 16 --steps 5 --warmup 3 --no-cpu-baseline --optimizer sgd > gpurun_out/rag_densenet_sgd.log 2>&1; echo "rc=$?" >> gpurun_out/rag_densenet_sgd.log
timeout 600 python bench.py --model resnet50 --batch 32 --steps 5 --warmup 3 --no-cpu-baseline --optimizer sgd > gpurun_out/rag_r50_sgd.log 2>&1; echo "rc=$?" >> gpurun_out/rag_r50_sgd.log
