#!/bin/bash
for e in 8 12; do echo "split EMU=$e $(TRACE_GAUSS=1 ./scripts/micro/attn_trace_$e | head -1)"; echo "noxch EMU=$e $(TRACE_GAUSS=1 ./scripts/micro/attn_noxch_$e | head -1)"; done
TRACE_GAUSS=1 ./scripts/micro/attn_noxch_8 | sed -n 8,14p
