#!/bin/bash
for r in 1 2; do for e in 8 12 16; do echo "deg3 EMU=$e $(TRACE_GAUSS=1 ./scripts/micro/attn_d3_$e | head -1)"; echo "deg2 EMU=$e $(TRACE_GAUSS=1 ./scripts/micro/attn_d2_$e | head -1)"; done; done
