timeout 600 python bench.py --steps 16 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/de.log 2>&1
python -c "
import json
for l in open('gpurun_out/de.log'):
    if l.startswith('{'):
        d=json.loads(l); print(d["value"], d["per_step_ms"]); print(d["host_phase_ms_fwd_bwd_step"]); print(d["allocator_in_region"])
" > gpurun_out/de_sum.log
