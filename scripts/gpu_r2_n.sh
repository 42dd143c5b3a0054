#!/bin/bash
# K1 per-f-chunk H readiness: parity, shard sizes, full C3/C5.
mkdir -p gpurun_out
OUT=gpurun_out/r2n.txt; : > $OUT
timeout 900 python -m pytest tests -m gpu -q -x -k "ffn or full_shape or variants or sharded" > gpurun_out/pytest_n.log 2>&1; tail -1 gpurun_out/pytest_n.log >> $OUT
for spec in "ffn_8b 1024" "ffn_8b 2048" "ffn_8b 4096" "ffn_8b 8192" "ffn_70b 4096" "ffn_70b 32768"; do
  set -- $spec
  echo "== $1 rows=$2" >> $OUT
  timeout 300 python bench.py --workload $1 --rows $2 --steps 20 --warmup 5 --no-cpu-baseline --no-adapter --no-check 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['value'],1), round(d['ms_per_step'],4), d['clocks']['sm_mhz'], d['clocks']['reasons'])" >> $OUT
done
cat $OUT
