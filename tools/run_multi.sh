# multi-GPU: parity check (fp32 + bf16) then the bench at N = number of visible GPUs
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
for m in fp32 bf16; do
  MATH=$m ROUNDS=4 timeout -s KILL 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511 tools/multi_gpu_check.py > gpurun_out/multi_$m.log 2>&1
  echo "multi $m exit $?"; grep -E "round|CHECK" gpurun_out/multi_$m.log | tail -5
done
timeout -s KILL 240 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus $N --steps ${STEPS:-2000} --warmup 10 > gpurun_out/bench_n$N.json 2> gpurun_out/bench_n$N.err
echo "bench n$N exit $?"; tail -3 gpurun_out/bench_n$N.err
python -c "
import json;d=json.load(open('gpurun_out/bench_n$N.json'));print('N', d['n_gpus'], d['value'], d['ms_per_step'], d.get('clocks'))"
for m in fp32 bf16; do
  PS_MODE=per_message MATH=$m ROUNDS=4 timeout -s KILL 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29521 tools/multi_gpu_check.py > gpurun_out/multi_pm_$m.log 2>&1
  echo "multi per-message $m exit $?"; grep -E "round|CHECK" gpurun_out/multi_pm_$m.log | tail -5
done
for m in fp32 bf16; do
  REPLAY=global MATH=$m ROUNDS=4 timeout -s KILL 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29531 tools/multi_gpu_check.py > gpurun_out/multi_gr_$m.log 2>&1
  echo "multi global-replay $m exit $?"; grep -E "round|CHECK" gpurun_out/multi_gr_$m.log | tail -6
done
timeout -s KILL 240 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29532 bench.py --gpus $N --steps ${STEPS:-2000} --warmup 10 --replay global --cpu-seconds 0 > gpurun_out/bench_gr_n$N.json 2> gpurun_out/bench_gr_n$N.err
echo "bench global-replay n$N exit $?"; tail -3 gpurun_out/bench_gr_n$N.err
python -c "
import json;d=json.load(open('gpurun_out/bench_gr_n$N.json'));print('global replay N', d['n_gpus'], d['value'], d['ms_per_step'], d['e2e']['value'])"
