timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "c1 or graph or ragged" 2>&1 | tail -2
for kv in "GORILA_FUSE_SAMPLE=0" "X=1" "GORILA_FUSE_SAMPLE=0" "X=1"; do env $kv timeout 200 python tools/qbench.py --reps 2 2>&1 | tail -1; done
