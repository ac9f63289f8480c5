#!/bin/bash
# One full ncu capture of the kernels matching $KREGEX (demangled name) in a short bench run.
mkdir -p gpurun_out
ARGS="--steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 2 ${EXTRA:-}"
python bench.py $ARGS > gpurun_out/ncu_plain.json 2> gpurun_out/ncu_plain.err && \
ncu --set full --metrics ${NCU_METRICS:-sm__ops_path_tensor_op_utchmma_src_bf16_dst_fp32.sum,l1tex__data_pipe_tc_wavefronts_mem_shared_op_utcmma_matrix_a.sum,l1tex__data_pipe_tc_wavefronts_mem_shared_op_utcmma_matrix_b_scope_1cta.sum,sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_elapsed} --clock-control none --import-source on --kernel-name-base demangled -k regex:"${KREGEX}" \
    -s ${SKIP:-10} -c ${COUNT:-2} -o gpurun_out/${OUT:-prof} -f python bench.py $ARGS > gpurun_out/ncu_full.log 2>&1
echo "ncu exit $?"
