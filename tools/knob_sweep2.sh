# B=32: weight-gradient split caps x cluster cap (same box)
mkdir -p gpurun_out
run() {
  env $1 timeout -s KILL 300 python bench.py --steps 4000 --warmup 5 --cpu-seconds 0 --capacity 200000 > gpurun_out/knob.json 2>gpurun_out/knob.err || { echo "$1 failed"; return; }
  python -c "
import json;d=json.load(open('gpurun_out/knob.json'));print('$1', round(d['value']), round(d['ms_per_step']*1000,2))"
}
for a in 16 8 6 4 11; do run "GORILA_WSPLIT_MAX=$a"; done
for b in 8 24 12; do run "GORILA_WSPLIT_MAX=8 GORILA_WSPLIT1_MAX=$b"; done
run "GORILA_WSPLIT_MAX=8 GORILA_CLUSTER_MAX=16"
run "GORILA_WSPLIT_MAX=6 GORILA_CLUSTER_MAX=16"
run "GORILA_WSPLIT_MAX=16"
