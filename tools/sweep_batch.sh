# configs[3]: per-GPU batch sweep on 1 GPU (1M-frame replay); one CSV row per batch into $OUT
OUT=${OUT:-gpurun_out/sweep_batch.csv}
mkdir -p gpurun_out
echo "batch,updates_per_s,frames_per_s,ms_per_step,step_tflops,roofline_kernel,roofline_frac" > $OUT
for b in ${BATCHES:-32 64 128 256 512 1024 2048 4096}; do
  steps=$(( b <= 256 ? 1000 : (b <= 1024 ? 300 : 100) ))
  timeout -s KILL 300 python bench.py --batch $b --steps $steps --warmup 5 --no-cpu-baseline --e2e-steps 5 > gpurun_out/sw_$b.json 2> gpurun_out/sw_$b.err
  python - $b >> $OUT <<'PY'
import json, sys
b = int(sys.argv[1])
d = json.load(open(f"gpurun_out/sw_{b}.json"))
tfl = 68.263936e6 * b * d["value"] / b / 1e12 * b  # algorithmic FLOP per update x updates/s
print(f"{b},{d['value']:.1f},{d['frames_per_s']:.0f},{d['ms_per_step']:.4f},{68.263936e6 * b * d['value'] / 1e12:.1f},"
      f"{d['roofline']['kernel']},{d['roofline']['frac']:.3f}")
PY
done
cat $OUT
