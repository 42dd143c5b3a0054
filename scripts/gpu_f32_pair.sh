#!/bin/bash
# fp32 GEMMs: CTA-pair 256x256 tiles (default where >= 148 tiles) vs the 128x256 single-CTA tiles
for rep in 1 2; do
  for v in 0 1; do echo "PAIR=$v"; BFGPU_F32_PAIR=$v timeout 200 python scripts/fp32_modes.py 2>&1 | head -2; done
done
