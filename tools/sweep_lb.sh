#!/bin/bash
for b in 32 256; do timeout 120 python tools/qbench.py --batch $b --steps 1000 --reps 2 --capacity 100000 2>&1 | tail -1; done
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "large_batch or c1" 2>&1 | tail -2
