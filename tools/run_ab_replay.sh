# global replay cost breakdown at N = visible GPUs: local / global / global without the barrier
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
run() {  # name, env, args
  env $2 timeout -s KILL 240 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29600 + RANDOM % 100)) bench.py --gpus $N --steps ${STEPS:-3000} --warmup 10 --cpu-seconds 0 $3 > gpurun_out/ab_$1.json 2> gpurun_out/ab_$1.err
  python -c "
import json;d=json.load(open('gpurun_out/ab_$1.json'));print('$1', round(d['value']), round(d['ms_per_step']*1000,1), 'us  e2e', round(d['e2e']['value']))"
}
run local "X=1" ""
run global "X=1" "--replay global"
run global_nobar "GORILA_REPLAY_BARRIER=0" "--replay global"
run local2 "X=1" "--learners 2 --capacity 200000"
run global2 "X=1" "--learners 2 --capacity 200000 --replay global"
