#!/bin/bash
# Full ncu capture (with source) of the kernels matching $KREGEX in a qbench run at batch $B; exports
# the raw metrics and the details page as CSV and the per-SASS-line source page of each kernel, then
# deletes the report (gpurun_out must stay small).
mkdir -p gpurun_out
B=${B:-4096}; OUT=${OUT:-deep}
python tools/qbench.py --batch $B --steps 20 --reps 1 --capacity 100000 > gpurun_out/${OUT}_plain.log 2>&1 || exit 1
ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k regex:"${KREGEX}" \
    -s ${SKIP:-0} -c ${COUNT:-3} -o /tmp/${OUT} -f python tools/qbench.py --batch $B --steps 3 --reps 1 --capacity 100000 \
    > gpurun_out/${OUT}_ncu.log 2>&1
ncu -i /tmp/${OUT}.ncu-rep --page raw --csv > gpurun_out/${OUT}_raw.csv
ncu -i /tmp/${OUT}.ncu-rep --page details --csv > gpurun_out/${OUT}_details.csv
N=$(python - <<PY
import csv,io,subprocess
o=subprocess.run(["ncu","-i","/tmp/${OUT}.ncu-rep","--page","raw","--csv"],capture_output=True,text=True).stdout
print(len(list(csv.reader(io.StringIO(o))))-2)
PY
)
for i in $(seq 0 $((N-1))); do
  ncu -i /tmp/${OUT}.ncu-rep --page source --csv --print-source ${PSRC:-cuda,sass} --launch-skip $i --launch-count 1 > gpurun_out/${OUT}_src$i.csv 2>&1
done
ls -la gpurun_out/ | grep ${OUT}
