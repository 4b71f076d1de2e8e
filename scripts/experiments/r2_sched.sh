#!/bin/bash
# inverse update schedule: next-row-only eager updates with fused pending K (default) vs the
# round-2 eager-rows schedule (SPDKFAC_EAGER_ROWS=1): parity, isolated inverse, bench
export PYTHONPATH=. SPD_WATCHDOG=900
timeout 900 python -m pytest tests/test_gpu_linalg.py tests/test_gpu_production_paths.py -m gpu -q -p no:cacheprovider -k "inverse or pivot or damped or small" > gpurun_out/r2_sched_tests.log 2>&1
echo "tests rc=$?"; tail -1 gpurun_out/r2_sched_tests.log; grep -E "^E  |FAILED|d=4608|d=2048" gpurun_out/r2_sched_tests.log | head
for v in 0 1; do
  SPDKFAC_EAGER_ROWS=$v timeout 300 python scripts/bench_inverse.py > gpurun_out/r2_inv_iso_er$v.json 2>&1; echo "inv er=$v rc=$?"
  python -c "
import json;d=json.load(open('gpurun_out/r2_inv_iso_er$v.json'))
for k,v in d.items():
  if isinstance(v,dict): print('er=$v', k, v['ms_total'], {c:(x['ms'],x['launches'],x['us_per_launch']) for c,x in v['cats'].items()})
" || tail -5 gpurun_out/r2_inv_iso_er$v.json
done
for v in 0 1; do
SPDKFAC_EAGER_ROWS=$v timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/r2_sched_bench$v.json 2>gpurun_out/r2_sched_bench$v.err
python -c "import json;d=json.loads(open('gpurun_out/r2_sched_bench$v.json').read().strip().splitlines()[-1]);print('bench er=$v', d['value'], {k:(v['kernel_ms_per_step'], v['frac']) for k,v in d['roofline_kernels'].items()})" || tail -5 gpurun_out/r2_sched_bench$v.err
done
timeout 900 python -m pytest tests/test_gpu_config_parity.py -m gpu -q -x -s -p no:cacheprovider > gpurun_out/r2_sched_cfg.log 2>&1
echo "cfg rc=$?"; tail -1 gpurun_out/r2_sched_cfg.log; grep worst gpurun_out/r2_sched_cfg.log
