#!/bin/bash
# One round of every kernel at batch $B under ncu --set full + the tcgen05 counters (qbench, after
# its warm-up rounds: -s skips the fill and the first rounds), raw page exported, report deleted.
mkdir -p gpurun_out
B=${B:-4096}; OUT=${OUT:-round$B}
python tools/qbench.py --batch $B --steps 20 --reps 1 --capacity 100000 > gpurun_out/${OUT}_plain.log 2>&1 || exit 1
ncu --set full --metrics sm__ops_path_tensor_op_utchmma_src_bf16_dst_fp32.sum,l1tex__data_pipe_tc_wavefronts_mem_shared_op_utcmma_matrix_a.sum,l1tex__data_pipe_tc_wavefronts_mem_shared_op_utcmma_matrix_b_scope_1cta.sum,sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_elapsed \
    --clock-control none --kernel-name-base demangled -k regex:"gorila::" -s ${SKIP:-300} -c ${COUNT:-19} -o /tmp/${OUT} -f \
    python tools/qbench.py --batch $B --steps 25 --reps 1 --capacity 100000 > gpurun_out/${OUT}_ncu.log 2>&1
ncu -i /tmp/${OUT}.ncu-rep --page raw --csv > gpurun_out/${OUT}_raw.csv
python tools/ncu_summary.py gpurun_out/${OUT}_raw.csv > gpurun_out/${OUT}_summary.txt
tail -25 gpurun_out/${OUT}_summary.txt
