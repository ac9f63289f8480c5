#!/bin/bash
# the -m gpu suite, then the batch points of the sweep with per-phase isolated times
mkdir -p gpurun_out
bash tools/gpu_tests.sh | tail -4
for b in ${BS:-4096 1024 256 32}; do timeout 300 python tools/qbench.py --batch $b --steps ${STEPS:-300} --reps 2 --capacity 100000 \
    --phases ${PH:-sample,conv1_fwd,conv2_fwd,conv3_fwd,fc4_fwd,fc4_dgrad,conv3_dgrad,conv2_dgrad,conv1_wgrad,conv2_wgrad,conv3_wgrad,fc4_wgrad,bias_grad} 2>&1 | tail -2; done
