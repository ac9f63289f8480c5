timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "replay or c1" 2>&1 | tail -2
timeout 300 python tools/qbench.py --batch 4096 --steps 30 --reps 2 --phases sample 2>&1 | tail -2
timeout 300 python tools/qbench.py --steps 3000 --reps 2 --phases sample 2>&1 | tail -2
