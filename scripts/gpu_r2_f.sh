#!/bin/bash
# Round 2 session re-entry: full GPU suite, smoke, every workload's bench line.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/gpu.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q -rf --durations=15 > gpurun_out/pytest_f.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke_f.log 2>&1
for w in ffn_8b lnmm_c1 lnmm attn ffn_70b; do
  timeout 900 python bench.py --workload $w --steps 20 --warmup 5 > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err
done
tail -25 gpurun_out/pytest_f.log
cat gpurun_out/smoke_f.log | tail -2
