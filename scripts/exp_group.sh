mkdir -p gpurun_out
for g in 4 8 16 32 64; do
  echo "group $g: $(BFGPU_FFN_GROUP=$g timeout 120 python scripts/quick_perf.py ffn 2>&1 | tr '\n' ' ')"
done
for g in 8 16 64; do
  BFGPU_FFN_GROUP=$g timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed -k regex:ffn_swiglu -s 2 -c 1 python scripts/ncu_target.py ffn_8b fused 3 2>&1 | grep -E "dram__|gpu__time|tensor" | sed "s/^/g=$g /"
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:ln_matmul -s 2 -c 1 -o gpurun_out/prof_lnmm -f python scripts/ncu_target.py lnmm fused 3 > gpurun_out/ncu_lnmm.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_kernel -s 2 -c 1 -o gpurun_out/prof_attn -f python scripts/ncu_target.py attn fused 3 > gpurun_out/ncu_attn.log 2>&1
