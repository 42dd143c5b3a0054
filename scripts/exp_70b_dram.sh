#!/bin/bash
M="dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum"
for pt in "8,9" "4,18" "16,4" "6,12"; do
  echo "== two_phase patch=$pt"
  BFGPU_FFN_PATCH=$pt timeout 300 ncu --metrics $M --clock-control none -k regex:ffn_swiglu -s 2 -c 2 --csv python scripts/ncu_target.py ffn_70b two_phase 2 2>/dev/null | grep -E 'dram__bytes|gpu__time' | awk -F'","' '{print $(NF-2), $(NF-1), $NF}'
done
timeout 120 python -m pytest tests/test_variants_gpu.py -q -k ffn 2>&1 | tail -1
