# quick GPU iteration: parity tests, then B=32 and large-batch benches (logs in gpurun_out/)
mkdir -p gpurun_out
timeout -s KILL 600 python -m pytest tests -m gpu -q -x --timeout 200 > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log; tail -15 gpurun_out/pytest_gpu.log
for b in ${BATCHES:-32 4096}; do
  timeout -s KILL 300 python bench.py --batch $b --capacity 200000 --steps ${STEPS:-300} --warmup 5 --cpu-seconds 0 > gpurun_out/bench_b$b.json 2> gpurun_out/bench_b$b.err
  echo "b$b exit $?"; tail -2 gpurun_out/bench_b$b.err
  python -c "
import json;d=json.load(open('gpurun_out/bench_b$b.json'));print($b, d['value'], d['ms_per_step'], {k: round(v,1) for k,v in (d.get('phases_isolated_us') or {}).items()})"
done
if [ -n "$AB_ENV" ]; then
  for b in ${AB_BATCHES:-4096}; do
    env $AB_ENV timeout -s KILL 300 python bench.py --batch $b --capacity 200000 --steps ${STEPS:-300} --warmup 5 --cpu-seconds 0 > gpurun_out/bench_ab_b$b.json 2> gpurun_out/bench_ab_b$b.err
    echo "AB($AB_ENV) b$b exit $?"; tail -2 gpurun_out/bench_ab_b$b.err
    python -c "
import json;d=json.load(open('gpurun_out/bench_ab_b$b.json'));print('AB', $b, d['value'], d['ms_per_step'], {k: round(v,1) for k,v in (d.get('phases_isolated_us') or {}).items()})"
  done
fi
