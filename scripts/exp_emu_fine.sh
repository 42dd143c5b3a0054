#!/bin/bash
for r in 1 2 3; do for e in 4 6 8 10; do echo "EMU=$e $(TRACE_GAUSS=1 ./scripts/micro/attn_e$e | head -1)"; done; done
