#!/bin/bash
# fc4 orientation switch (GORILA_FC4_NORMAL_MIN) at the sweep's middle batches
for b in 256 512 1024 2048; do for nm in 256 100000; do
  GORILA_FC4_NORMAL_MIN=$nm timeout 300 python tools/qbench.py --batch $b --steps 300 --reps 2 --capacity 100000 --phases fc4_fwd,fc4_dgrad 2>&1 | tail -2 | tr '\n' ' '; echo
done; done
