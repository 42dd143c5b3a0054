#!/bin/bash
timeout 600 python -m pytest tests/test_ffn_gpu.py tests/test_variants_gpu.py -x -q 2>&1 | tail -2
for i in 1 2 3; do timeout 120 python scripts/quick_perf.py ffn 2>&1 | grep K1; done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:ffn_swiglu -s 2 -c 1 -o gpurun_out/prof_ffn -f python scripts/ncu_target.py ffn_8b fused 3 > gpurun_out/ncu_ffn.log 2>&1
tail -1 gpurun_out/ncu_ffn.log
timeout 300 python bench.py --workload ffn_70b --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('C5', d['value'], d['clocks'])"
