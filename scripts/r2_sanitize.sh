#!/bin/bash
# compute-sanitizer over the operator-level GPU tests (one tool per call: memcheck or racecheck),
# against the sanitizer build of the library (mbarrier watchdog raised; `make -C
# paper_2107_06533_b200/csrc sanitize`).  Usage: bash scripts/r2_sanitize.sh memcheck|racecheck
TOOL=${1:-memcheck}
export PYTHONPATH=. SPDKFAC_LIB=$PWD/paper_2107_06533_b200/lib/libspdkfac_sanitize.so
mkdir -p gpurun_out
SEL="not 4608 and not 2304 and not 2048 and not production and not config and not bert and not many_rows"
timeout 2400 compute-sanitizer --tool $TOOL --error-exitcode 17 --print-limit 50 --target-processes all \
  python -m pytest tests/test_gpu_linalg.py tests/test_gpu_optimizer.py -m gpu -q -x -p no:cacheprovider \
  -k "$SEL" > gpurun_out/r2_sanitize_$TOOL.log 2>&1
echo "rc=$?" >> gpurun_out/r2_sanitize_$TOOL.log
tail -15 gpurun_out/r2_sanitize_$TOOL.log
