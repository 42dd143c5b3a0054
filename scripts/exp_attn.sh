#!/bin/bash
for r in 1 2; do for st in 0 200 400 800; do echo "stagger=$st $(TRACE_GAUSS=1 ./scripts/micro/attn_st_$st | head -1)"; done; done
