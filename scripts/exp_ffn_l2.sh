#!/bin/bash
# K1 L2 policy / group sweep: time (quick_perf) and DRAM bytes per launch (ncu) at C3 and C5.
mkdir -p gpurun_out
for h in 0 1; do for g in 16 32 64; do
  echo "hints=$h group=$g"
  BFGPU_FFN_L2HINTS=$h BFGPU_FFN_GROUP=$g timeout 120 python scripts/quick_perf.py ffn 2>&1 | grep fused
  BFGPU_FFN_L2HINTS=$h BFGPU_FFN_GROUP=$g timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:ffn_swiglu -s 2 -c 1 --csv python scripts/ncu_target.py ffn_8b fused 3 2>/dev/null | grep -E 'dram__bytes|gpu__time' | awk -F'","' '{print $(NF-2), $(NF-1), $NF}'
done; done
