#!/bin/bash
# K3 split-softmax variant: parity with BFGPU_ATTN_SPLIT=1, then A/B against the ping-pong kernel.
mkdir -p gpurun_out
BFGPU_ATTN_SPLIT=1 timeout 600 python -m pytest tests/test_attention_gpu.py tests/test_full_shape_gpu.py -k "attention or attn or c2 or golden or shapes or extreme" -q -x -rf > gpurun_out/pytest_split.log 2>&1
tail -5 gpurun_out/pytest_split.log
for rep in 1 2 3; do
  for sp in 0 1; do
    r=$(BFGPU_ATTN_SPLIT=$sp timeout 300 python bench.py --workload attn --steps 20 --warmup 5 --no-cpu-baseline --no-adapter --no-check 2>gpurun_out/b_err_$sp.txt | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['value'],1), round(d['ms_per_step'],4), d['clocks']['sm_mhz'], d['plan']['kernel'])")
    echo "split=$sp $r"
  done
done
BFGPU_ATTN_SPLIT=1 timeout 300 python scripts/quick_perf.py attn
