#!/bin/bash
timeout 600 python -m pytest tests/test_ffn_gpu.py tests/test_lnmm_gpu.py tests/test_attention_gpu.py -x -q 2>&1 | tail -1
for r in 1 2; do timeout 200 python scripts/quick_perf.py 2>&1 | grep -E "^K|SDPA|cuBLAS"; done
