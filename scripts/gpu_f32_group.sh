#!/bin/bash
# fp32-mode tile raster group sweep (BFGPU_F32_GROUP) at the C3/C4/C1 shapes
for g in 2 4 8 16; do echo "group $g"; BFGPU_F32_GROUP=$g timeout 200 python scripts/fp32_modes.py 2>&1 | head -2; done
echo "default"; timeout 200 python scripts/fp32_modes.py 2>&1 | head -2
python scripts/c1_breakdown.py
