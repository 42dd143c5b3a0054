#!/bin/bash
# K1 at C3: cross-cluster sync and group under burst and sustained timing.
for rep in 1 2; do
  for cfg in "BFGPU_NOP=1" "BFGPU_FFN_WAVESYNC=1" "BFGPU_FFN_GROUP=64" "BFGPU_FFN_SEGSYNC=0"; do
    r=$(env $cfg timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-adapter --no-check --sustained-s 2 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); s=d['sustained']; print(round(d['value'],1), 'sus', round(s['value'],1), s['clocks']['sm_mhz'], d['plan']['sync'], d['plan']['group'])")
    echo "$cfg $r"
  done
done
