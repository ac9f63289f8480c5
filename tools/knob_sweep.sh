# B=32 step under each launch-shape knob (same box): value, us/step, isolated fc4 phases
mkdir -p gpurun_out
for kv in "X=1" "GORILA_CLUSTER_MAX=16" "GORILA_CLUSTER_MAX=4" "GORILA_WSPLIT_MAX=32" "GORILA_WSPLIT_MAX=8" "GORILA_FC4_NORMAL_MIN=1" "GORILA_FORK=0" "GORILA_PDL=0" "X=2"; do
  env $kv timeout -s KILL 300 python bench.py --steps 3000 --warmup 5 --cpu-seconds 0 --capacity 200000 > gpurun_out/knob.json 2>gpurun_out/knob.err || { echo "$kv failed"; tail -3 gpurun_out/knob.err; continue; }
  python -c "
import json;d=json.load(open('gpurun_out/knob.json'));p=d['phases_isolated_us'];print('$kv', round(d['value']), round(d['ms_per_step']*1000,2), {k: round(p[k],1) for k in ('fc4_fwd','fc4_dgrad','fc4_wgrad','fc5_fwd','wgrad_reduce','conv1_wgrad')})"
done
