#!/bin/bash
# K1 scheduling group at shard sizes: the planner's L2-derived group vs the schedule model's pick.
for rep in 1 2; do
  for cfg in "2048 16" "2048 8" "2048 4" "4096 32" "4096 16" "1024 8" "1024 4"; do
    set -- $cfg
    r=$(BFGPU_FFN_GROUP=$2 timeout 300 python bench.py --rows $1 --steps 20 --warmup 5 --no-cpu-baseline --no-adapter --no-check --sustained-s 0 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['value'],1), d['plan']['group'], round(d['plan']['sched_eff'],3))")
    echo "rows=$1 group128=$2 $r"
  done
done
