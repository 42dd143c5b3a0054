#!/bin/bash
timeout 300 python -m pytest tests/test_attention_gpu.py tests/test_from_host_gpu.py -x -q 2>&1 | tail -1
timeout 300 python -m pytest tests/test_variants_gpu.py -x -q -k attn 2>&1 | tail -1
for r in 1 2 3; do for e in 8 12; do echo "EMU=$e"; BFGPU_ATTN_EMU=$e timeout 120 python scripts/quick_perf.py attn 2>&1 | grep -v "^$"; done; done
TRACE_GAUSS=1 ./scripts/micro/attn_trace_8 | sed -n 1,16p
