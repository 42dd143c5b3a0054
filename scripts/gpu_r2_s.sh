#!/bin/bash
mkdir -p gpurun_out
BFGPU_ATTN_WS=1 timeout 900 python -m pytest tests -m gpu -q -x -rf -k "attention or attn or c2 or snapshot or concurrency" > gpurun_out/pytest_s.log 2>&1
tail -3 gpurun_out/pytest_s.log
for rep in 1 2 3; do
  for ws in 0 1; do
    r=$(BFGPU_ATTN_WS=$ws timeout 300 python bench.py --workload attn --steps 20 --warmup 5 --no-cpu-baseline --no-adapter --no-check 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['value'],1), round(d['ms_per_step'],4), d['clocks']['sm_mhz'])")
    echo "ws=$ws $r"
  done
done
