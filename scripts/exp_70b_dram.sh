#!/bin/bash
M="dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum"
for ws in 0 1; do for sch in fused two_phase; do
  echo "== wavesync=$ws $sch"
  BFGPU_FFN_WAVESYNC=$ws timeout 300 ncu --metrics $M --clock-control none -k regex:ffn_swiglu -s 2 -c 2 --csv python scripts/ncu_target.py ffn_70b $sch 2 2>/dev/null | grep -E 'dram__bytes|gpu__time' | awk -F'","' '{print $(NF-2), $(NF-1), $NF}'
done; done
for ws in 0 1; do WHICH=fused BFGPU_FFN_WAVESYNC=$ws timeout 300 python scripts/exp_70b.py 2>&1 | grep TFLOP; BFGPU_FFN_WAVESYNC=$ws timeout 200 python scripts/quick_perf.py ffn 2>&1 | grep fused; done
BFGPU_FFN_WAVESYNC=1 timeout 300 python -m pytest tests/test_ffn_gpu.py -q -x 2>&1 | tail -1
