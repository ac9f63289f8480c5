#!/bin/bash
# Per-launch device times of one bench configuration (cold-cache, serialised: compare shares).
mkdir -p gpurun_out
ARGS="--steps ${STEPS:-40} --warmup 3 --no-cpu-baseline --e2e-steps 3 ${EXTRA:-}"
python bench.py $ARGS > gpurun_out/ncu_plain.json 2> gpurun_out/ncu_plain.err && \
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'gemm|k_' -c ${COUNT:-800} --csv \
    --log-file gpurun_out/launches.csv python bench.py $ARGS > gpurun_out/ncu.log 2>&1
echo "ncu exit $?"
python tools/summarize_launches.py gpurun_out/launches.csv
