TAG=b32 bash tools/bench_run.sh | tail -3
TAG=b4096 BENCH_ARGS="--batch 4096 --steps 30 --warmup 5" bash tools/bench_run.sh | tail -3
B=4096 bash tools/ncu_round.sh > /dev/null 2>&1; B=32 SKIP=600 bash tools/ncu_round.sh > /dev/null 2>&1
ls gpurun_out | grep round
