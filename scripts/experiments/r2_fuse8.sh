#!/bin/bash
# kFuse 8 vs 4: inverse parity (subset), isolated inverse, bench
export PYTHONPATH=. SPD_WATCHDOG=900
for lib in libspdkfac_fuse8.so libspdkfac.so; do
  export SPDKFAC_LIB=paper_2107_06533_b200/lib/$lib
  timeout 600 python -m pytest tests/test_gpu_linalg.py tests/test_gpu_production_paths.py -m gpu -q -p no:cacheprovider -k "damped" > gpurun_out/r2_f8_tests_$lib.log 2>&1
  echo "$lib tests rc=$?"; tail -1 gpurun_out/r2_f8_tests_$lib.log
  timeout 300 python scripts/bench_inverse.py > gpurun_out/r2_inv_iso_$lib.json 2>&1
  python -c "
import json;d=json.load(open('gpurun_out/r2_inv_iso_$lib.json'))
for k,v in d.items():
  if isinstance(v,dict): print('$lib', k, v['ms_total'], {c:(x['ms'],x['launches'],x['us_per_launch']) for c,x in v['cats'].items()})
" || tail -5 gpurun_out/r2_inv_iso_$lib.json
  timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/r2_f8_bench_$lib.json 2>gpurun_out/r2_f8_bench_$lib.err
  python -c "import json;d=json.loads(open('gpurun_out/r2_f8_bench_$lib.json').read().strip().splitlines()[-1]);print('bench $lib', d['value'], {k:(v['kernel_ms_per_step'], v['frac']) for k,v in d['roofline_kernels'].items()})" || tail -5 gpurun_out/r2_f8_bench_$lib.err
done
