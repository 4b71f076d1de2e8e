timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29541 -m paper_2107_06533_b200.calibrate --out gpurun_out/b200_p2.params > gpurun_out/calib_p2.log 2>&1
echo "rc=$?" >> gpurun_out/calib_p2.log
