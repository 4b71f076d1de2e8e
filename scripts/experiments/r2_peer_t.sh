#!/bin/bash
export PYTHONPATH=.
timeout 420 python -m pytest tests/test_gpu_multi.py -m gpu -q -k "peer and 2" -p no:cacheprovider -s > gpurun_out/peer_tests.log 2>&1
echo "tests rc=$?"; tail -c 6000 gpurun_out/peer_tests.log
