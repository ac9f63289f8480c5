# A/B of two library builds on the same box: libgorila_old.so (GORILA_LIB) vs the in-tree build
mkdir -p gpurun_out
for rep in 1 2; do
for lib in old new; do
  if [ $lib = old ]; then export GORILA_LIB=$PWD/paper_1507_04296_b200/libgorila_old.so; else unset GORILA_LIB; fi
  timeout -s KILL 300 python bench.py --steps ${STEPS:-3000} --warmup 5 --cpu-seconds 0 --capacity 200000 ${BENCH_ARGS} > gpurun_out/ab_lib_$lib.json 2>/dev/null
  python -c "
import json;d=json.load(open('gpurun_out/ab_lib_$lib.json'));print('$lib', round(d['value']), round(d['ms_per_step']*1000,2), 'e2e', round(d['e2e']['value']))"
done
done
