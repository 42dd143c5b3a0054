#!/bin/bash
for g in ${GLIST:-16 8 32 16 8 32 12 24}; do
  BFGPU_LNMM_GROUP=$g timeout 300 python bench.py --workload lnmm --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('group $g', round(d['value'],1))"
done
