#!/bin/bash
mkdir -p gpurun_out
BFGPU_ATTN_Q1=${Q1:-0} timeout 120 ./scripts/micro/attn_trace > gpurun_out/attn_trace_new.txt 2>&1
cat gpurun_out/attn_trace_new.txt
