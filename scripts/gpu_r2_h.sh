#!/bin/bash
# K1: L2 policy (evict-first weights, evict-last X/H) + discard, by group size; ncu DRAM bytes.
mkdir -p gpurun_out
OUT=gpurun_out/r2h.txt; : > $OUT
for cfg in "1 1 32" "1 1 16" "1 1 8" "0 1 16" "1 0 8"; do
  set -- $cfg
  echo "== C3 hints=$1 discard=$2 group128=$3" >> $OUT
  BFGPU_FFN_HINTS=$1 BFGPU_FFN_DISCARD=$2 BFGPU_FFN_GROUP=$3 timeout 120 python scripts/quick_perf.py ffn 2>&1 | grep fused >> $OUT
  BFGPU_FFN_HINTS=$1 BFGPU_FFN_DISCARD=$2 BFGPU_FFN_GROUP=$3 timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:ffn_swiglu -s 2 -c 1 --csv python scripts/ncu_target.py ffn_8b fused 3 2>/dev/null | grep -E 'dram__bytes|gpu__time|lts__' | awk -F'","' '{print $(NF-2), $(NF-1), $NF}' >> $OUT
done
BFGPU_FFN_HINTS=1 timeout 300 python -m pytest tests/test_full_shape_gpu.py -q -x -k "c3" >> $OUT 2>&1
cat $OUT
