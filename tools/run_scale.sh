# the driver's scaling series on one box: N = 1, 2, 4 (as many as visible), bench lines into gpurun_out/scale_n*.json
mkdir -p gpurun_out
NG=$(nvidia-smi -L | wc -l)
CUDA_VISIBLE_DEVICES=0 timeout -s KILL 300 python bench.py > gpurun_out/scale_n1.json 2> gpurun_out/scale_n1.err
echo "n1 exit $?"
for n in 2 4; do
  [ $n -le $NG ] || continue
  timeout -s KILL 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29700+n)) bench.py --gpus $n > gpurun_out/scale_n$n.json 2> gpurun_out/scale_n$n.err
  echo "n$n exit $?"
done
for n in 1 2 4; do [ -s gpurun_out/scale_n$n.json ] && python -c "
import json; d=json.load(open('gpurun_out/scale_n$n.json')); print($n, round(d['value']), round(d['ms_per_step']*1000, 2), 'e2e', round(d['e2e']['value']), d['roofline']['kernel'], round(d['roofline']['frac'], 3), d['clocks'])"; done
