#!/bin/bash
mkdir -p gpurun_out
for ks in 1 2; do
  BFGPU_FFN_KSPLIT=$ks timeout 600 ncu --set full --clock-control none --import-source on -k regex:ffn_swiglu -s 2 -c 1 -o gpurun_out/prof_ffn1024_ks$ks -f python scripts/ncu_ffn_rows.py 1024 3 > gpurun_out/ncu_ffn1024_ks$ks.log 2>&1
  BFGPU_FFN_KSPLIT=$ks timeout 600 ncu --set full --clock-control none -k regex:ffn_swiglu -s 2 -c 1 -o gpurun_out/prof_ffn8192_ks$ks -f python scripts/ncu_ffn_rows.py 8192 3 > gpurun_out/ncu_ffn8192_ks$ks.log 2>&1
done
ls -la gpurun_out/*.ncu-rep
