export SPD_WATCHDOG=250
for i in 1 2; do
(cd _ab_old && timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > ../gpurun_out/x_old.log 2>&1)
python -c "
import json
for l in open('gpurun_out/x_old.log'):
    if l.startswith('{'):
        d=json.loads(l); print('old', d['value'])
" >> gpurun_out/x_sum.log
timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/x_new.log 2>&1
python -c "
import json
for l in open('gpurun_out/x_new.log'):
    if l.startswith('{'):
        d=json.loads(l); print('new', d['value'])
" >> gpurun_out/x_sum.log
done
