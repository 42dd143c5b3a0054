#!/bin/bash
timeout 600 python -m pytest tests/test_ffn_gpu.py tests/test_variants_gpu.py -x -q -k "ffn" 2>&1 | tail -1
for r in 1 2 3; do for sv in 1 0; do
  BFGPU_FFN_SEGSYNC=$sv timeout 300 python bench.py --workload ffn_8b --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('segsync $sv', round(d['value'],1))"
done; done
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__cycles_elapsed.avg.per_second
for sv in 1 0; do echo "segsync $sv"; BFGPU_FFN_SEGSYNC=$sv timeout 300 ncu --metrics $M --clock-control none -k regex:ffn_swiglu -s 2 -c 1 --csv python scripts/ncu_target.py ffn_8b fused 3 2>/dev/null | grep -E '"(gpu__|sm__|dram__)' | awk -F'","' '{print $(NF-2), $NF}'; done
