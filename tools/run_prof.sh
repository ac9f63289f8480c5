# parity + benches (run_quick.sh), then one ncu --set full capture (tools/ncu_full.sh) if they passed
bash tools/run_quick.sh && grep -q "pytest exit 0" gpurun_out/pytest_gpu.log && bash tools/ncu_full.sh
