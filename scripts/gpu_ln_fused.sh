#!/bin/bash
# K2 fp32: one launch (split folded into the GEMM) vs split + GEMM, at C1 (warm graph replay) and C4
for rep in 1 2; do
  for f in 0 1; do
    echo "LN_FUSED=$f $(BFGPU_F32_LN_FUSED=$f python scripts/c1_breakdown.py | tail -1)"
    BFGPU_F32_LN_FUSED=$f timeout 200 python scripts/fp32_modes.py 2>&1 | sed -n 2p
  done
done
