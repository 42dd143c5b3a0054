#!/bin/bash
# K3 FMA-pipe exponential split under burst and sustained (power-capped) timing.
for rep in 1 2; do
  for e in 0 8 12 16; do
    r=$(BFGPU_ATTN_EMU=$e timeout 300 python bench.py --workload attn --steps 20 --warmup 5 --no-cpu-baseline --no-adapter --no-check --sustained-s 2 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); s=d['sustained']; print(round(d['value'],1), 'sus', round(s['value'],1), s['clocks']['sm_mhz'])")
    echo "emu=$e $r"
  done
done
