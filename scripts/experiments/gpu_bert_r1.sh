#!/bin/bash
# configs[4]: BERT-base linears through SPD-KFAC (parity test + N=1 bench, SGD floor beside it).
mkdir -p gpurun_out
export SPD_WATCHDOG=400
timeout 600 python -m pytest tests/test_gpu_optimizer.py -q -x -k token > gpurun_out/bert_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/bert_pytest.log
timeout 600 python bench.py --model bert_base_linears --steps 10 --warmup 3 > gpurun_out/bert_bench.json 2> gpurun_out/bert_bench.err
timeout 300 python bench.py --model bert_base_linears --optimizer sgd --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bert_sgd.json 2> gpurun_out/bert_sgd.err
tail -3 gpurun_out/bert_pytest.log; cut -c1-250 gpurun_out/bert_bench.json gpurun_out/bert_sgd.json; tail -5 gpurun_out/bert_bench.err
