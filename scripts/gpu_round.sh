#!/bin/bash
# One GPU session: tests, smoke, bench lines, launch list, ncu captures of the kernels.
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err
for w in attn lnmm ffn_70b; do timeout 300 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err; done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_under_ncu.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_attn.csv python bench.py --workload attn --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_attn_under_ncu.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_kernel -s 2 -c 1 -o gpurun_out/prof_attn -f python scripts/ncu_target.py attn fused 3 > gpurun_out/ncu_attn.log 2>&1
if [ "$FULL" = 1 ]; then
timeout 600 ncu --set full --clock-control none --import-source on -k regex:ffn_swiglu -s 2 -c 1 -o gpurun_out/prof_ffn -f python scripts/ncu_target.py ffn_8b fused 3 > gpurun_out/ncu_ffn.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:ln_matmul -s 2 -c 1 -o gpurun_out/prof_lnmm -f python scripts/ncu_target.py lnmm fused 3 > gpurun_out/ncu_lnmm.log 2>&1
fi
[ "$FULL" = 1 ] && timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/nvsmi.txt
true
if [ "$FULL" = 1 ]; then
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:ffn_swiglu -s 1 -c 1 -o gpurun_out/prof_ffn70b -f python scripts/ncu_target.py ffn_70b fused 2 > gpurun_out/ncu_ffn70b.log 2>&1
fi
