#!/bin/bash
for g in 32 64 128 256; do WHICH=fused BFGPU_FFN_GROUP=$g timeout 300 python scripts/exp_70b.py 2>&1 | grep TFLOP; done
