#!/bin/bash
# one gpurun call: the -m gpu suite (logs + junit under gpurun_out/)
mkdir -p gpurun_out
export GORILA_CONTEXT_OUT=gpurun_out/context_bf16_vs_exact.json
timeout ${T:-2400} python -m pytest tests -m gpu -q -x ${ARGS:-} -rs --junitxml=gpurun_out/gputest.xml > gpurun_out/gputest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/gputest.log
tail -30 gpurun_out/gputest.log
