#!/bin/bash
# default bench line + launch list (+ optional extra bench args), results under gpurun_out/
mkdir -p gpurun_out
TAG=${TAG:-b32}
timeout ${T:-900} python bench.py ${BENCH_ARGS:-} > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err
echo "bench rc=$?"; cat gpurun_out/bench_${TAG}.json | head -c 3000; echo
if [ -n "$LAUNCHES" ]; then
  STEPS=40 bash tools/ncu_launches.sh > gpurun_out/launches_${TAG}.txt 2>&1; tail -40 gpurun_out/launches_${TAG}.txt
fi
