#!/bin/bash
# GPU-box check: tests, smoke, short bench. Everything under timeouts; logs in gpurun_out/.
mkdir -p gpurun_out
( nvidia-smi; nproc; lscpu | grep -i "model name" ) > gpurun_out/box.txt 2>&1
timeout -s KILL 900 python -m pytest tests -m gpu -q --timeout 300 > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout -s KILL 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1
echo "smoke exit $?" >> gpurun_out/smoke.log
timeout -s KILL 600 python bench.py --steps ${BENCH_STEPS:-300} --warmup 5 --cpu-seconds 10 > gpurun_out/bench.json 2> gpurun_out/bench.err
echo "bench exit $?" >> gpurun_out/bench.err
tail -3 gpurun_out/pytest_gpu.log; tail -2 gpurun_out/smoke.log; cat gpurun_out/bench.json | head -c 3000; tail -5 gpurun_out/bench.err
