#!/bin/bash
M="dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum"
for ws in 0 1; do
  echo "== wavesync=$ws"
  for i in 1 2; do BFGPU_FFN_WAVESYNC=$ws BFGPU_LNMM_WAVESYNC=$ws timeout 200 python scripts/quick_perf.py ffn lnmm 2>&1 | grep -E 'fused|K2:'; done
  BFGPU_LNMM_WAVESYNC=$ws timeout 300 ncu --metrics $M --clock-control none -k regex:ln_matmul -s 2 -c 1 --csv python scripts/ncu_target.py lnmm fused 3 2>/dev/null | grep -E 'dram__bytes' | awk -F'","' '{print $(NF-2), $(NF-1), $NF}'
  BFGPU_FFN_WAVESYNC=$ws timeout 300 ncu --metrics $M --clock-control none -k regex:ffn_swiglu -s 2 -c 1 --csv python scripts/ncu_target.py ffn_8b fused 3 2>/dev/null | grep -E 'dram__bytes' | awk -F'","' '{print $(NF-2), $(NF-1), $NF}'
done
BFGPU_LNMM_WAVESYNC=1 timeout 300 python -m pytest tests/test_lnmm_gpu.py -q -x 2>&1 | tail -1
