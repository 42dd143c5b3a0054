#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -x -rf -k "c1 or fp32 or f32 or lnmm" > gpurun_out/pytest_c1.log 2>&1; tail -2 gpurun_out/pytest_c1.log
for rep in 1 2 3; do timeout 300 python bench.py --workload lnmm_c1 --steps 50 --warmup 10 --no-cpu-baseline --no-adapter 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['value'],2), round(d['ms_per_step']*1000,2), 'us', d['check']['pass'])"; done
