#!/bin/bash
# on an N-GPU box: the -m gpu multi-rank tests (one rank per GPU via NCCL + the one-GPU ipc variants), then the
# scaling series N = 1, 2, 4 of the default bench (as many as visible) and the async bench across GPUs
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_multi.py -q -x -rs > gpurun_out/multi_tests.log 2>&1; echo "multi tests rc=$?"; tail -4 gpurun_out/multi_tests.log
bash tools/run_scale.sh
NG=$(nvidia-smi -L | wc -l)
timeout -s KILL 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29761 \
   bench.py --gpus $NG --ps-mode async --learners 4 --capacity 200000 --steps 300 --warmup 5 --max-staleness 2 --no-cpu-baseline \
   > gpurun_out/bench_async_n$NG.json 2> gpurun_out/bench_async_n$NG.err; echo "async n$NG rc=$?"
python -c "
import json; d=json.loads(open('gpurun_out/bench_async_n$NG.json').read().strip().splitlines()[-1]); a=d['async']
print('async', d['n_gpus'], round(d['value']), 'fresh', a['fresh_per_shard'], 'stale', a['stale_per_shard'], 'rej', a['rejected_outlier'])"
