#!/bin/bash
# Round 2 check: full -m gpu suite, then the default N=1 bench line, and the same with the
# round-1 FFMA pivot sweep (SPDKFAC_PIVOT=ffma) for an A/B of the pivot kernel.
mkdir -p gpurun_out
export PYTHONPATH=.
timeout 1500 python -m pytest tests -m gpu -q -s -p no:cacheprovider > gpurun_out/r2_gpu.log 2>&1
echo "rc=$?" >> gpurun_out/r2_gpu.log
tail -3 gpurun_out/r2_gpu.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r2_bench.json 2> gpurun_out/r2_bench.err
echo "bench rc=$?"
SPDKFAC_PIVOT=ffma timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/r2_bench_ffma.json 2>/dev/null
python - <<'PY'
import json
for f in ("gpurun_out/r2_bench.json", "gpurun_out/r2_bench_ffma.json"):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        print(f, d["value"], (d.get("e2e") or {}).get("value"), {k: v["ms_per_step"] for k, v in d["kernel_breakdown"].items() if isinstance(v, dict)})
        print("  roofline", json.dumps(d.get("roofline")))
        print("  iteration", json.dumps(d.get("iteration_roofline")))
        print("  peaks", json.dumps(d.get("peaks_measured")), "cpu", json.dumps(d.get("cpu_baseline")))
    except Exception as e:
        print(f, "ERR", e)
PY
