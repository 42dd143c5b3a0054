#!/bin/bash
for r in 1 2 3; do for pl in 0 1 2; do echo "place $pl $(TRACE_GAUSS=1 ./scripts/micro/attn_place_$pl | head -1)"; done; done
