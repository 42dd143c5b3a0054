#!/bin/bash
# K1 with direct epilogue stores and a 7th operand stage (variants/libbfgpu_direct.so) vs the default.
L=paper_2505_07829_b200/lib/libbfgpu.so
cp $L /tmp/intree.so
cp variants/libbfgpu_direct.so $L
timeout 900 python -m pytest tests/test_ffn_gpu.py tests/test_full_shape_gpu.py -q -x -k "ffn or c3 or c5 or ragged" 2>&1 | tail -2
cp /tmp/intree.so $L
for rep in 1 2 3; do
  for v in base direct; do
    cp variants/libbfgpu_$v.so $L
    r=$(timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-adapter --no-check 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); s=d['sustained']; print(round(d['value'],1), 'sustained', round(s['value'],1), s['clocks']['sm_mhz'])")
    echo "$v $r"
  done
done
cp /tmp/intree.so $L
