timeout 600 python -m pytest tests/test_ffn_gpu.py tests/test_variants_gpu.py -x -q -k "ffn or FFN" 2>&1 | tail -1
for r in 1 2; do
for w in ffn_70b ffn_8b; do timeout 300 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$w', round(d['value'],1), d['clocks']['sm_mhz'])"; done
done
