#!/bin/bash
# u8 staging: parity of the large-batch paths, then the batch sweep
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_large_batch.py tests/test_gpu_parity.py tests/test_gpu_act.py -q -x -m gpu \
    -k "large_batch or ragged or act" 2>&1 | tail -5
for b in ${BS:-4096 1024 256 128 32}; do timeout 300 python tools/qbench.py --batch $b --steps ${STEPS:-200} --reps 2 --capacity 100000 \
    --phases sample,conv1_fwd,conv1_wgrad 2>&1 | tail -2; done
