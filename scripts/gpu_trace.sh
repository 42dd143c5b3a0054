#!/bin/bash
mkdir -p gpurun_out
timeout 120 ./scripts/micro/attn_trace > gpurun_out/attn_trace_new.txt 2>&1
cat gpurun_out/attn_trace_new.txt
