#!/bin/bash
# Round-1 re-entry check: GPU parity tests, smoke, N=1 bench (both arms) on a fresh box.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/fin_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/fin_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/fin_smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/fin_bench.json 2> gpurun_out/fin_bench.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/fin_ref.json 2> gpurun_out/fin_ref.err
tail -3 gpurun_out/fin_pytest.log; tail -1 gpurun_out/fin_smoke.log; cut -c1-300 gpurun_out/fin_bench.json; cut -c1-300 gpurun_out/fin_ref.json
