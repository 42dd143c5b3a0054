#!/bin/bash
timeout 300 python -m pytest tests/test_attention_gpu.py -x -q 2>&1 | tail -1
for r in 1 2 3 4; do echo "old $(TRACE_GAUSS=1 ./scripts/micro/attn_old_8 | head -1)"; echo "new $(TRACE_GAUSS=1 ./scripts/micro/attn_trace_8 | head -1)"; done
for r in 1 2; do timeout 120 python scripts/quick_perf.py attn 2>&1 | grep -v "^$"; done
