#!/bin/bash
# K1 H-line discard A/B at C3/C5 (time + ncu DRAM bytes), group sizes; 8-GPU shard sizes on one GPU.
mkdir -p gpurun_out
OUT=gpurun_out/r2g.txt; : > $OUT
timeout 600 python -m pytest tests -m gpu -q -x -k "ffn" > gpurun_out/pytest_g.log 2>&1; tail -1 gpurun_out/pytest_g.log >> $OUT
for cfg in "1 32" "0 32" "1 16" "0 16" "1 8"; do
  set -- $cfg
  echo "== C3 discard=$1 group128=$2" >> $OUT
  BFGPU_FFN_DISCARD=$1 BFGPU_FFN_GROUP=$2 timeout 120 python scripts/quick_perf.py ffn 2>&1 | grep fused >> $OUT
  BFGPU_FFN_DISCARD=$1 BFGPU_FFN_GROUP=$2 timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:ffn_swiglu -s 2 -c 1 --csv python scripts/ncu_target.py ffn_8b fused 3 2>/dev/null | grep -E 'dram__bytes|gpu__time' | awk -F'","' '{print $(NF-2), $(NF-1), $NF}' >> $OUT
done
for d in 1 0; do
  echo "== C5 discard=$d" >> $OUT
  BFGPU_FFN_DISCARD=$d timeout 300 python bench.py --workload ffn_70b --steps 10 --warmup 3 --no-cpu-baseline --no-adapter --no-check 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['clocks'])" >> $OUT
  BFGPU_FFN_DISCARD=$d timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:ffn_swiglu -s 1 -c 1 --csv python scripts/ncu_target.py ffn_70b fused 2 2>/dev/null | grep -E 'dram__bytes|gpu__time' | awk -F'","' '{print $(NF-2), $(NF-1), $NF}' >> $OUT
done
for spec in "ffn_8b 1024" "ffn_8b 2048" "ffn_8b 4096" "ffn_70b 4096" "ffn_70b 8192" "lnmm 8192" "attn 32"; do
  set -- $spec
  echo "== shard $1 rows=$2" >> $OUT
  timeout 300 python bench.py --workload $1 --rows $2 --steps 20 --warmup 5 --no-cpu-baseline --no-adapter --no-check 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['clocks']['sm_mhz'])" >> $OUT
done
cat $OUT
