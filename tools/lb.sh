KREGEX="gemm|k_conv_tower|k_sample|k_apply|k_fc5|k_bias|k_wgrad" EXTRA="--batch 4096 --capacity 100000 --e2e-steps 2" SKIP=40 COUNT=20 OUT=b4096 bash tools/ncu_full.sh
python tools/ncu_summary.py gpurun_out/b4096.ncu-rep > gpurun_out/b4096_summary.txt; cat gpurun_out/b4096_summary.txt
KREGEX="gemm|k_conv_tower|k_sample|k_apply|k_fc5|k_bias|k_wgrad|k_pack" EXTRA="--e2e-steps 2" SKIP=100 COUNT=17 OUT=b32 bash tools/ncu_full.sh
python tools/ncu_summary.py gpurun_out/b32.ncu-rep > gpurun_out/b32_summary.txt; cat gpurun_out/b32_summary.txt
