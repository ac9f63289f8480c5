set -x
which nvidia-smi nvidia-cuda-mps-control
nvidia-smi -L
nvidia-smi -q -d CLOCK | head -40
nproc; grep -m1 "model name" /proc/cpuinfo
ncu --query-metrics --chip gb100 > gpurun_out/ncu_metrics_gb100.txt 2>&1
ncu --query-metrics-mode suffix --metrics sm__pipe_tensor_op_umma_cycles_active,sm__inst_executed_pipe_umma --chip gb100 > gpurun_out/ncu_metrics_suffix.txt 2>&1
grep -i "umma\|tensor\|tmem\|utc" gpurun_out/ncu_metrics_gb100.txt | head -80
