#!/bin/bash
# Multi-GPU re-run after the fp16-plane inverse (N GPUs): calibration at P = N, NCCL parity tests,
# bench with the fitted params (e2e), and the D-KFAC / MPD-KFAC baselines.
N=${1:-2}
export PYTHONPATH=. SPD_WATCHDOG=900
mkdir -p gpurun_out
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
timeout 900 $TR --master-port 29611 -m paper_2107_06533_b200.calibrate --out gpurun_out/b200_p$N.params > gpurun_out/r2b_calib_p$N.log 2>&1
echo "calibrate rc=$?"; grep -E "batched|wrote" gpurun_out/r2b_calib_p$N.log | tail -3
timeout 1200 python -m pytest tests/test_gpu_multi.py -m gpu -q -p no:cacheprovider > gpurun_out/r2b_multi_tests_p$N.log 2>&1
echo "multi tests rc=$?"; tail -2 gpurun_out/r2b_multi_tests_p$N.log
run() {  # name, extra flags
  timeout 900 $TR --master-port $((29620 + RANDOM % 300)) bench.py --gpus $N --steps 20 --warmup 5 $2 > gpurun_out/r2b_bench_n${N}_$1.json 2> gpurun_out/r2b_bench_n${N}_$1.err
  python -c "import json;d=json.loads(open('gpurun_out/r2b_bench_n${N}_$1.json').read().strip().splitlines()[-1]);print('$1', d['value'], (d.get('e2e') or {}).get('value'), 'nct', d.get('placement_nct_tensors'), 'busbw', (d.get('peaks_measured') or {}).get('nccl_allreduce_busbw_gbs'))" || tail -3 gpurun_out/r2b_bench_n${N}_$1.err
}
run fitted "--perf-params gpurun_out/b200_p$N.params"
run default ""
for sch in mpdkfac dkfac; do run $sch "--scheme $sch --perf-params gpurun_out/b200_p$N.params --no-e2e"; done
