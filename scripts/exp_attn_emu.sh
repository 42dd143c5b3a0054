timeout 600 python -m pytest tests/test_attention_gpu.py tests/test_variants_gpu.py tests/test_from_host_gpu.py -x -q -k "attn or attention or from_host or K3 or c2 or golden or shapes or extreme" 2>&1 | tail -1
timeout 600 python -m pytest tests/test_attention_gpu.py tests/test_variants_gpu.py -x -q 2>&1 | tail -1
for r in 1 2; do for e in 8 12 16; do echo "EMU=$e"; BFGPU_ATTN_EMU=$e timeout 120 python scripts/quick_perf.py attn 2>&1 | grep -v "^$"; done; done
