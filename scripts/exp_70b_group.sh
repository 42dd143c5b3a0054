#!/bin/bash
# C5 group-size sweep with the wave sync on (its default at this size): short bench runs
for g in ${GLIST:-64 16 128 32 16 64 32 8}; do
  BFGPU_FFN_GROUP=$g timeout 300 python bench.py --workload ffn_70b --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('group $g', round(d['value'],1), d['clocks']['sm_mhz'])"
done
