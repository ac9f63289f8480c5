# N-GPU bench A/B over env settings (device-timed value only); usage: bash tools/run_ab_multi.sh "ENV1" "ENV2" ...
N=$(nvidia-smi -L | wc -l)
mkdir -p gpurun_out
i=0
for e in "$@"; do
  env $e timeout -s KILL 240 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29600+i)) bench.py --gpus $N --steps 2000 --warmup 10 --no-cpu-baseline --e2e-steps 20 > gpurun_out/ab_$i.json 2> gpurun_out/ab_$i.err
  echo "[$e] exit $?: $(python -c "import json;d=json.load(open('gpurun_out/ab_$i.json'));print(d['value'], d['ms_per_step'])" 2>&1 | tail -1)"
  i=$((i+1))
done
