#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -rf -k "fp32 or f32 or c1 or concurrency" > gpurun_out/pytest_q.log 2>&1
tail -3 gpurun_out/pytest_q.log
timeout 300 python bench.py --workload lnmm_c1 --steps 50 --warmup 5 --no-cpu-baseline --no-adapter > gpurun_out/bench_c1_v2.json 2> gpurun_out/bench_c1_v2.err
python -c "import json; d=json.loads(open('gpurun_out/bench_c1_v2.json').read().strip().splitlines()[-1]); print(round(d['value'],2), round(d['ms_per_step']*1e3,1), 'us', d['check']['rel'], d['plan']['grid'], d['plan']['resident_ctas'])"
timeout 300 ncu --set full --clock-control none --import-source on -k regex:"f32x3|f32_split" -s 4 -c 2 -o gpurun_out/prof_c1_v2 -f python scripts/ncu_target.py lnmm_c1 fused 4 > gpurun_out/ncu_c1_v2.log 2>&1
tail -1 gpurun_out/ncu_c1_v2.log
