mkdir -p gpurun_out
run() {
  env $1 timeout -s KILL 300 python bench.py --steps 4000 --warmup 5 --cpu-seconds 0 --capacity 200000 $2 > gpurun_out/knob.json 2>gpurun_out/knob.err || { echo "$1 failed"; tail -2 gpurun_out/knob.err; return; }
  python -c "
import json;d=json.load(open('gpurun_out/knob.json'));print('$1 $2', round(d['value']), round(d['ms_per_step']*1000,2))"
}
run "X=1"
for c in 444 592 888; do run "GORILA_SIDE_RED_CTAS=$c"; done
