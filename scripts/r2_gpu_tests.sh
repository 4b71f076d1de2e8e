#!/bin/bash
# Round 2: full -m gpu suite on one B200 (config-level parity prints per-layer errors with -s).
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -s -p no:cacheprovider --timeout 1500 ${PYTEST_ARGS} > gpurun_out/r2_gpu.log 2>&1
echo "rc=$?" >> gpurun_out/r2_gpu.log
tail -4 gpurun_out/r2_gpu.log
