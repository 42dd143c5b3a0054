#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "fp32 or f32 or c1 or execute or cli" > gpurun_out/pytest_b.log 2>&1
timeout 600 python bench.py --workload lnmm_c1 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err
timeout 900 python bench.py --workload ffn_8b --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_ffn8b_b.json 2> gpurun_out/bench_ffn8b_b.err
tail -2 gpurun_out/pytest_b.log
