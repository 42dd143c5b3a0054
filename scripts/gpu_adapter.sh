#!/bin/bash
for w in ffn_8b lnmm ffn_70b; do
  timeout 600 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline --no-check --sustained-s 0 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); a=d['e2e_adapter']; print('$w', round(a['value'],2), a['ms_per_call'], a['stages_ms_best_call'])"
done
nproc
