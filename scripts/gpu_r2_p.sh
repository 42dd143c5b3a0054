#!/bin/bash
mkdir -p gpurun_out
for v in base chunk; do
  cp variants/libbfgpu_$v.so paper_2505_07829_b200/lib/libbfgpu.so
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:ffn_swiglu -s 2 -c 1 -o gpurun_out/prof_k1_$v -f python scripts/ncu_target.py ffn_8b fused 3 > gpurun_out/ncu_k1_$v.log 2>&1
  tail -1 gpurun_out/ncu_k1_$v.log
done
