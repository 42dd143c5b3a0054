#!/bin/bash
for e in 0 4 8 12; do echo "EMU=$e $(BFGPU_ATTN_EMU=$e timeout 120 python scripts/quick_perf.py attn 2>&1 | grep K3)"; done
