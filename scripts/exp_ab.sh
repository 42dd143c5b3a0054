#!/bin/bash
# A/B of the K1 wave sync at C3 plus a K3 pipeline trace
for r in 1 2 3; do
  for w in 1 0; do echo "wavesync=$w"; BFGPU_FFN_WAVESYNC=$w timeout 120 python scripts/quick_perf.py ffn 2>&1 | grep K1; done
done
timeout 120 python scripts/quick_perf.py lnmm attn 2>&1 | grep -v "^$"
./scripts/micro/attn_trace_0 > gpurun_out/trace_base.txt 2>&1
TRACE_GAUSS=1 ./scripts/micro/attn_trace_0 > gpurun_out/trace_gauss.txt 2>&1
nvidia-smi --query-gpu=clocks.sm,power.draw,temperature.gpu --format=csv
