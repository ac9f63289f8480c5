#!/bin/bash
# A/B of the shipped library against paper_1507_04296_b200/libgorila_exp.so (a variant build) at $BS
for lib in libgorila.so libgorila_exp.so; do for b in ${BS:-4096}; do
  GORILA_LIB=paper_1507_04296_b200/$lib timeout 300 python tools/qbench.py --batch $b --steps ${STEPS:-200} --reps 2 --capacity 100000 --phases ${PH:-conv1_fwd} 2>&1 | tail -2
done; done
