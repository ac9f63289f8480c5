#!/bin/bash
for b in 2048; do
  for kv in "GORILA_PDL=1" "GORILA_PDL=0"; do
    env $kv timeout 120 python tools/qbench.py --batch $b --steps 40 --reps 2 --capacity 100000 2>&1 | tail -1
  done
done
