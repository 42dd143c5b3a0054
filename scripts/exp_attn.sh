#!/bin/bash
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_attention_gpu.py -x -q > gpurun_out/attn_tests.log 2>&1
tail -3 gpurun_out/attn_tests.log
for i in 1 2; do timeout 120 python scripts/quick_perf.py attn 2>&1; done
TRACE_GAUSS=1 ./scripts/micro/attn_trace_0 | tail -12
