#!/bin/bash
# K3 study: phase trace, quick_perf vs SDPA, ncu full capture with source of the current kernel.
mkdir -p gpurun_out
timeout 120 ./scripts/micro/attn_trace > gpurun_out/attn_trace.txt 2>&1
TRACE_GAUSS=1 timeout 120 ./scripts/micro/attn_trace > gpurun_out/attn_trace_gauss.txt 2>&1
timeout 300 python scripts/quick_perf.py attn > gpurun_out/qp_attn.txt 2>&1
timeout 300 python scripts/quick_perf.py attn >> gpurun_out/qp_attn.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_kernel -s 2 -c 1 -o gpurun_out/prof_attn -f python scripts/ncu_target.py attn fused 3 > gpurun_out/ncu_attn.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:sdpa -s 2 -c 1 -o gpurun_out/prof_sdpa -f python scripts/ncu_sdpa.py > gpurun_out/ncu_sdpa.log 2>&1
cat gpurun_out/attn_trace.txt gpurun_out/qp_attn.txt
