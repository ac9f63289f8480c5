#!/bin/bash
# scaling series with the fused GEMM + reduce-scatter (push) and without (GORILA_PUSH=0: owners pull)
mkdir -p gpurun_out
NG=$(nvidia-smi -L | wc -l)
for mode in push pull; do
  envs=""; [ $mode = pull ] && envs="GORILA_PUSH=0"
  for n in 2 4; do
    [ $n -le $NG ] || continue
    env $envs timeout -s KILL 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
       --master-port $((29800+n)) bench.py --gpus $n --steps 2000 --e2e-steps 300 > gpurun_out/scale_${mode}_n$n.json 2> gpurun_out/scale_${mode}_n$n.err
    python -c "
import json; d=json.load(open('gpurun_out/scale_${mode}_n$n.json')); print('$mode', $n, round(d['value']), round(d['ms_per_step']*1000, 2), 'e2e', round(d['e2e']['value']), d['clocks']['sm_mhz'])" || tail -3 gpurun_out/scale_${mode}_n$n.err
  done
done
