#!/bin/bash
mkdir -p gpurun_out
for g in 2 4 8 16 32; do echo "group=$g"
BFGPU_LNMM_GROUP=$g timeout 120 python scripts/quick_perf.py lnmm 2>&1 | grep 'K2:'
BFGPU_LNMM_GROUP=$g timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:ln_matmul -s 2 -c 1 --csv python scripts/ncu_target.py lnmm fused 3 2>/dev/null | grep -E 'dram__bytes' | awk -F'","' '{print $(NF-2), $(NF-1), $NF}'
done
