#!/bin/bash
# fp32 GEMM tile width A/B (BFGPU_F32_BN=128 vs the default, 256 where tiles allow)
for rep in 1 2; do
  for bn in 128 256; do echo "BN $bn"; BFGPU_F32_BN=$bn timeout 200 python scripts/fp32_modes.py 2>&1 | head -2; done
done
python scripts/c1_breakdown.py
