#!/bin/bash
# K2 512x256 tiles: fused vs staged (statistics in their own launch) to isolate the statistics hand-off.
for rep in 1 2; do
  for sch in fused two_phase; do
    for w in 0 1; do
      r=$(BFGPU_LNMM_WIDE=$w timeout 300 python bench.py --workload lnmm --schedule $sch --steps 20 --warmup 5 --no-cpu-baseline --no-adapter --no-check --sustained-s 0 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['value'],1), round(d['ms_per_step'],4), d['plan']['kernel'])")
      echo "$sch wide=$w $r"
    done
  done
done
