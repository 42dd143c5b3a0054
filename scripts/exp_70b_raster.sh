#!/bin/bash
run() { env $1 timeout 300 python bench.py --workload ffn_70b --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$1', round(d['value'],1), d['clocks']['sm_mhz'])"; }
for r in 1 2; do
  run "BFGPU_FFN_GROUP=16"
  run "BFGPU_FFN_BRASTER=4"
  run "BFGPU_FFN_GROUP=32 BFGPU_FFN_BRASTER=8"
  run "BFGPU_FFN_GROUP=32 BFGPU_FFN_BRASTER=4"
done
