#!/bin/bash
mkdir -p gpurun_out
python scripts/c1_vendor.py > gpurun_out/c1_vendor.json 2>&1; cat gpurun_out/c1_vendor.json
