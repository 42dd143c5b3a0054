mkdir -p gpurun_out
timeout 120 python scripts/quick_ffn.py 2>&1 | grep -v Warning | tail -20
timeout 200 python -m pytest tests/test_ffn_gpu.py -q --tb=line -x 2>&1 | tail -5
echo "2SM:"; timeout 120 python scripts/quick_perf.py ffn
echo "1SM:"; BFGPU_FFN_1SM=1 timeout 120 python scripts/quick_perf.py ffn
for g in 16 64; do echo "2SM group $g: $(BFGPU_FFN_GROUP=$g timeout 120 python scripts/quick_perf.py ffn 2>&1 | tr '\n' ' ')"; done
