#!/bin/bash
for g in ${GLIST:-32 16 32 16 24 32}; do
  BFGPU_FFN_GROUP=$g timeout 300 python bench.py --workload ffn_8b --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('group $g', round(d['value'],1))"
done
