#!/bin/bash
# Measured unfused baselines: timing, then per-step DRAM bytes of every kernel under ncu.
mkdir -p gpurun_out
timeout 300 python scripts/unfused_baseline.py time > gpurun_out/unfused_time.jsonl 2> gpurun_out/unfused_time.err
for w in ffn_8b lnmm attn; do
  timeout 600 ncu --profile-from-start off --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/unfused_$w.csv python scripts/unfused_baseline.py ncu $w > gpurun_out/unfused_ncu_$w.log 2>&1
done
# fused kernels' dram bytes with the same metric set (for a like-for-like column)
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:bfgpu -s 2 -c 3 --csv --log-file gpurun_out/fused_dram.csv python scripts/ncu_target.py ffn_8b fused 3 > /dev/null 2>&1
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:bfgpu -s 2 -c 3 --csv --log-file gpurun_out/fused_dram_lnmm.csv python scripts/ncu_target.py lnmm fused 3 > /dev/null 2>&1
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:bfgpu -s 2 -c 3 --csv --log-file gpurun_out/fused_dram_attn.csv python scripts/ncu_target.py attn fused 3 > /dev/null 2>&1
cat gpurun_out/unfused_time.jsonl
