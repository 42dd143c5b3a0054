#!/bin/bash
for sv in 1 0 1 0; do echo "segsync $sv"; BFGPU_FFN_SEGSYNC=$sv timeout 300 python scripts/exp_power.py ffn 2>&1 | tail -1; done
