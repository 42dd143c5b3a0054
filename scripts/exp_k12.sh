#!/bin/bash
timeout 600 python -m pytest tests/test_ffn_gpu.py tests/test_lnmm_gpu.py -x -q 2>&1 | tail -2
for i in 1 2; do timeout 200 python scripts/quick_perf.py ffn lnmm 2>&1 | grep -E 'fused|K2:'; done
