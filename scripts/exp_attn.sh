#!/bin/bash
# K3: parity tests, timing per exp-emulation split.
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_attention_gpu.py -x -q > gpurun_out/attn_tests.log 2>&1
tail -3 gpurun_out/attn_tests.log
for e in 0 8 12 16; do echo "EMU=$e"; BFGPU_ATTN_EMU=$e timeout 120 python scripts/quick_perf.py attn 2>&1 | grep -v SDPA; done
for e in 0 12 16; do TRACE_GAUSS=1 ./scripts/micro/attn_trace_$e | head -1; done
