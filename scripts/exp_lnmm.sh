timeout 300 python -m pytest tests/test_lnmm_gpu.py tests/test_ffn_gpu.py -q --tb=line -x 2>&1 | tail -3
timeout 100 python scripts/debug_bitwise.py 2>&1
echo "2SM:"; timeout 120 python scripts/quick_perf.py lnmm ffn 2>&1
echo "1SM:"; BFGPU_LNMM_1SM=1 timeout 120 python scripts/quick_perf.py lnmm 2>&1 | head -1
