#!/bin/bash
# each im2col case in its own process (an illegal instruction poisons the context)
export PYTHONPATH=.
for i in 0 1 2 3 4 5 6 7; do
  timeout 300 python -m pytest tests/test_gpu_production_paths.py -m gpu -q -p no:cacheprovider -k "im2col_tma_engine and 1-shape$i-" > gpurun_out/r2_i2c_case$i.log 2>&1
  echo "case $i rc=$? $(tail -1 gpurun_out/r2_i2c_case$i.log)"
done
timeout 300 python -m pytest tests/test_gpu_production_paths.py -m gpu -q -p no:cacheprovider -k "mixed" > gpurun_out/r2_i2c_mixed.log 2>&1; echo "mixed rc=$? $(tail -1 gpurun_out/r2_i2c_mixed.log)"
