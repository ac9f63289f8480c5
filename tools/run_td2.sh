bash tools/gpu_check.sh
for b in 256 1024 4096; do timeout -s KILL 300 python bench.py --batch $b --capacity 200000 --steps 30 --warmup 3 --cpu-seconds 0 > gpurun_out/bench_b$b.json 2> gpurun_out/bench_b$b.err; echo "b$b exit $?"; python -c "
import json;d=json.load(open('gpurun_out/bench_b$b.json'));print($b, d['value'], d['ms_per_step'], d.get('phases_isolated_us'))"; done
