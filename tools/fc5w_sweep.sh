# fc5 forward + TD at large batch: samples per warp (S) x warps per block, default heuristic first
for b in 256 1024 4096; do
  for kv in "X=0" "GORILA_FC5W_S=1 GORILA_FC5W_WARPS=16" "GORILA_FC5W_S=2 GORILA_FC5W_WARPS=8" "GORILA_FC5W_S=4 GORILA_FC5W_WARPS=4" "GORILA_FC5W_S=4 GORILA_FC5W_WARPS=8" "GORILA_FC5W_S=2 GORILA_FC5W_WARPS=4"; do
    env $kv timeout 200 python tools/qbench.py --batch $b --steps 200 --reps 2 --capacity 100000 --phases fc5_fwd 2>&1 | tail -2 | tr '\n' ' '; echo
  done
done
