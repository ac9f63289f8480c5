#!/bin/bash
# end-of-round evidence on one GPU: the -m gpu suite, smoke(), the default bench line and the B=4096 line
mkdir -p gpurun_out
bash tools/gpu_tests.sh | tail -3
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
TAG=final_b32 bash tools/bench_run.sh | tail -1 | head -c 300; echo
TAG=final_b4096 BENCH_ARGS="--batch 4096 --steps 30 --warmup 5" bash tools/bench_run.sh | tail -1 | head -c 300; echo
