#!/bin/bash
# fp32 mode of K2 on tcgen05 (3xTF32): parity tests, C1 bench vs the SIMT kernel, ncu of both launches.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -rf -k "fp32 or f32 or c1 or lnmm or execute or cli" > gpurun_out/pytest_j.log 2>&1
tail -5 gpurun_out/pytest_j.log
timeout 300 python bench.py --workload lnmm_c1 --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/bench_c1_x3.json 2> gpurun_out/bench_c1_x3.err
BFGPU_F32_SIMT=1 timeout 300 python bench.py --workload lnmm_c1 --steps 50 --warmup 5 --no-cpu-baseline --no-adapter > gpurun_out/bench_c1_simt.json 2> gpurun_out/bench_c1_simt.err
for f in bench_c1_x3 bench_c1_simt; do python -c "import json; d=json.loads(open('gpurun_out/$f.json').read().strip().splitlines()[-1]); print('$f', round(d['value'],2), round(d['ms_per_step']*1e3,1), 'us', d['gpu_launches'], d['check'], d.get('e2e',{}).get('value'))"; done
timeout 300 ncu --set full --clock-control none --import-source on -k regex:"f32x3|f32_split" -s 4 -c 2 -o gpurun_out/prof_c1 -f python scripts/ncu_target.py lnmm_c1 fused 4 > gpurun_out/ncu_c1.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c1.csv python bench.py --workload lnmm_c1 --steps 3 --warmup 3 --no-cpu-baseline --no-adapter --no-check > gpurun_out/bench_c1_under_ncu.log 2>&1
tail -2 gpurun_out/ncu_c1.log
