#!/bin/bash
# NEXT row f2 bench lines: N = 1 and N = 2 ranks on one GPU (ipc bootstrap), 4 learners per rank
mkdir -p gpurun_out
A="--ps-mode async --learners ${LRN:-4} --capacity 200000 --steps ${STEPS:-300} --warmup 5 --max-staleness ${MD:-4} --no-cpu-baseline"
timeout 600 python bench.py $A > gpurun_out/bench_async_n1.json 2> gpurun_out/bench_async_n1.err; echo "n1 rc=$?"
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 29877 \
    bench.py $A --gpus 2 --bootstrap ipc > gpurun_out/bench_async_n2.json 2> gpurun_out/bench_async_n2.err; echo "n2 rc=$?"
for f in gpurun_out/bench_async_n1.json gpurun_out/bench_async_n2.json; do
python -c "
import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); a=d['async']
print('$f', round(d['value']), 'updates/s', round(d['ms_per_step']*1000,1), 'us/step', 'sent', a['sent'], 'rejected', a['rejected_outlier'], 'fresh', a['fresh_per_shard'], 'stale', a['stale_per_shard'])" || tail -5 ${f%.json}.err
done
