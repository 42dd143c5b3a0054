#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_d.log 2>&1
timeout 600 python bench.py --workload lnmm_c1 --steps 50 --warmup 5 --no-cpu-baseline --no-adapter > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err
tail -15 gpurun_out/pytest_d.log
