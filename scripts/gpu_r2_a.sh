#!/bin/bash
# Round 2 session A: FP32 peak, fp32-mode parity, every workload's bench line with its CPU baseline.
mkdir -p gpurun_out
./scripts/micro/ffma_peak > gpurun_out/ffma_peak.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q -x -k "fp32 or f32 or c1 or generic or execute or cli" > gpurun_out/pytest_f32.log 2>&1
for w in lnmm_c1 attn lnmm ffn_70b ffn_8b; do
  timeout 900 python bench.py --workload $w --steps 10 --warmup 3 > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err
done
tail -2 gpurun_out/pytest_f32.log
