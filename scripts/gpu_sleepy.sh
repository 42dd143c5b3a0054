#!/bin/bash
L=paper_2505_07829_b200/lib/libbfgpu.so
cp $L /tmp/intree.so
for rep in 1 2; do
  for v in base sleepy500 sleepy2k; do
    cp variants/libbfgpu_$v.so $L
    for w in ffn_8b lnmm; do
      r=$(timeout 300 python bench.py --workload $w --steps 20 --warmup 5 --no-cpu-baseline --no-adapter --no-check --sustained-s 2 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); s=d['sustained']; print(round(d['value'],1), 'sus', round(s['value'],1), s['clocks']['sm_mhz'])")
      echo "$v $w $r"
    done
  done
done
cp /tmp/intree.so $L
