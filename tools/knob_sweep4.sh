mkdir -p gpurun_out
for rep in 1 2; do for v in 0 1 2 3; do GORILA_PDL_PREFETCH=$v python bench.py --steps 4000 --warmup 5 --cpu-seconds 0 --capacity 200000 > gpurun_out/knob.json 2>/dev/null; python -c "
import json;d=json.load(open('gpurun_out/knob.json'));p=d['phases_isolated_us'];print('prefetch $v', round(d['value']), round(d['ms_per_step']*1000,2), {k: round(p[k],1) for k in ('fc4_fwd','fc4_dgrad','conv3_dgrad','conv2_dgrad')})"; done; done
