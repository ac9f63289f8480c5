# fc5 / sampler changes: every GPU test, the fc5 phases, then the batch sweep
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for b in 4096 1024 256; do timeout 300 python tools/qbench.py --batch $b --steps 200 --reps 2 --capacity 100000 --phases sample,fc5_fwd,fc5_bwd 2>&1 | tail -2; done
BATCHES="${BATCHES:-32 64 128 256 512 1024 2048 4096}" OUT=gpurun_out/sweep_fc5.csv bash tools/sweep_batch.sh 2>&1 | tail -9
