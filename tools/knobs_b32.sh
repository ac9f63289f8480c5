for kv in "X=0" "GORILA_CLUSTER_MAX=16" "GORILA_CLUSTER_MAX=4" "GORILA_FC5_FUSE=1" "GORILA_SPLIT_REDUCE=0" "GORILA_WSPLIT1_MAX=8" "GORILA_WSPLIT1_MAX=32"; do
  env $kv timeout 200 python tools/qbench.py --batch 32 --steps 2000 --reps 3 --capacity 100000 2>&1 | tail -1
done
