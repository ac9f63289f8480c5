#!/bin/bash
# quick probe: the ipc bootstrap, N ranks sharing cuda:0
mkdir -p gpurun_out
N=${N:-2}
timeout ${T:-600} python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr 127.0.0.1 --master-port 29611 \
   tools/multi_gpu_check.py > gpurun_out/multi_${TAG:-x}.log 2>&1
echo "rc=$?" >> gpurun_out/multi_${TAG:-x}.log
tail -25 gpurun_out/multi_${TAG:-x}.log
