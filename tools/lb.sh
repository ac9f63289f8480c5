KREGEX="k_fc5" EXTRA="--batch 4096 --capacity 100000 --e2e-steps 2" SKIP=2 COUNT=4 OUT=fc5 bash tools/ncu_full.sh
python tools/ncu_summary.py gpurun_out/fc5.ncu-rep
ncu -i gpurun_out/fc5.ncu-rep --page details --csv 2>/dev/null | grep -i "warp cycles per issued\|Stall\|Issued Warp\|Achieved Occupancy\|Duration" | head -40
