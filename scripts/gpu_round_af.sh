export SPD_WATCHDOG=250
for i in 1 2; do
for w in old new; do
if [ $w = old ]; then cd _ab_old; else cd $GRAFT_REPO_ROOT; fi
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 2956$i bench.py --gpus 2 --steps 30 --warmup 3 --no-e2e --no-cpu-baseline > $GRAFT_REPO_ROOT/gpurun_out/af.log 2>&1
cd $GRAFT_REPO_ROOT
python -c "
import json
for l in open('gpurun_out/af.log'):
    if l.startswith('{'):
        d=json.loads(l); print('$w', d['value'])
" >> gpurun_out/af_sum.log
done
done
