#!/bin/bash
for r in 1 2 3; do for a in 2 4 8; do echo "ahead $a $(TRACE_GAUSS=1 ./scripts/micro/attn_pf$a | head -1)"; done; done
