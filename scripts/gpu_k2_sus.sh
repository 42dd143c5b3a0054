#!/bin/bash
# K2 at C4: scheduling group under burst and sustained timing.
for rep in 1 2; do
  for g in 16 8 32; do
    r=$(BFGPU_LNMM_GROUP=$g timeout 300 python bench.py --workload lnmm --steps 20 --warmup 5 --no-cpu-baseline --no-adapter --no-check --sustained-s 2 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); s=d['sustained']; print(round(d['value'],1), 'sus', round(s['value'],1), s['clocks']['sm_mhz'])")
    echo "group=$g $r"
  done
done
