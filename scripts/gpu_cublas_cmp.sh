#!/bin/bash
mkdir -p gpurun_out
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second,lts__t_sectors_srcunit_tex.sum,l1tex__m_xbar2l1tex_read_bytes.sum,launch__grid_size,launch__cluster_dim_x,launch__cluster_dim_y,launch__block_size,smsp__inst_executed.sum,launch__registers_per_thread"
timeout 300 ncu --metrics $M --clock-control none -k regex:"nvjet|gemm|cutlass|sm100" -c 2 --csv python scripts/ncu_cublas8k.py 2>/dev/null | grep -v "^==" > gpurun_out/cublas_cmp.csv
timeout 300 ncu --metrics $M --clock-control none -k regex:ffn_swiglu -s 2 -c 1 --csv python scripts/ncu_target.py ffn_8b fused 3 2>/dev/null | grep -v "^==" > gpurun_out/k1_cmp.csv

