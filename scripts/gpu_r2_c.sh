#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_sharded_gpu.py -q -x > gpurun_out/pytest_sharded.log 2>&1
timeout 600 python bench.py --workload lnmm_c1 --steps 50 --warmup 5 --no-cpu-baseline --no-adapter > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_f32 -s 2 -c 1 -o gpurun_out/prof_c1 -f python scripts/ncu_target.py lnmm_c1 fused 3 > gpurun_out/ncu_c1.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c1.csv python bench.py --workload lnmm_c1 --steps 3 --warmup 3 --no-cpu-baseline --no-adapter --no-check > gpurun_out/bench_c1_under_ncu.log 2>&1
tail -2 gpurun_out/pytest_sharded.log
