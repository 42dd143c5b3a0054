#!/bin/bash
# K3 one-query-tile variant (BFGPU_ATTN_Q1=1): parity, then A/B against the ping-pong kernel.
mkdir -p gpurun_out
BFGPU_ATTN_Q1=1 timeout 900 python -m pytest tests/test_attention_gpu.py tests/test_full_shape_gpu.py tests/test_concurrency_gpu.py -k "attention or attn or c2 or golden or shapes or extreme or concurr" -q -x -rf > gpurun_out/pytest_q1.log 2>&1
tail -3 gpurun_out/pytest_q1.log
for rep in 1 2 3; do
  for q in 0 1; do
    r=$(BFGPU_ATTN_Q1=$q timeout 300 python bench.py --workload attn --steps 20 --warmup 5 --no-cpu-baseline --no-adapter --no-check 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['value'],1), round(d['ms_per_step'],4), d['plan']['kernel'])")
    echo "q1=$q $r"
  done
done
BFGPU_ATTN_Q1=1 timeout 300 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second,lts__t_sectors_srcunit_tex.sum,dram__bytes_read.sum --clock-control none -k regex:attn -s 2 -c 1 --csv python scripts/ncu_target.py attn fused 3 2>/dev/null | grep -E 'gpu__time|tensor|per_second|srcunit|dram' | awk -F'","' '{print $(NF-2), $(NF-1), $NF}'
