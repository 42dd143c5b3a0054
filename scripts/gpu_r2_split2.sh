#!/bin/bash
# K3 split softmax with a MUFU token (BFGPU_ATTN_SPLIT=1): parity, then A/B against the ping-pong kernel.
mkdir -p gpurun_out
BFGPU_ATTN_SPLIT=1 timeout 600 python -m pytest tests/test_attention_gpu.py tests/test_full_shape_gpu.py tests/test_shape_sweep_gpu.py -k "attention or attn or c2 or golden or shapes or extreme" -q -x -rf > gpurun_out/pytest_split.log 2>&1
tail -3 gpurun_out/pytest_split.log
for rep in 1 2 3; do
  for sp in 0 1; do
    r=$(BFGPU_ATTN_SPLIT=$sp timeout 300 python bench.py --workload attn --steps 20 --warmup 5 --no-cpu-baseline --no-adapter --no-check --sustained-s 1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['value'],1), round(d['ms_per_step'],4), 'sus', round(d['sustained']['value'],1), d['plan']['kernel'])")
    echo "split=$sp $r"
  done
done
