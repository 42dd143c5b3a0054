#!/bin/bash
# Round-2 evidence (session 4, after the fp32-mode work): full GPU suite, smoke, every bench workload (with CPU baselines), the
# reference arm, launch lists and ncu --set full captures of each product kernel.
mkdir -p gpurun_out/final5
O=gpurun_out/final5
nvidia-smi --query-gpu=name,clocks.max.sm,power.limit --format=csv > $O/nvsmi.txt
timeout 1500 python -m pytest tests -m gpu -q -rf > $O/pytest_gpu.log 2>&1; tail -2 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1; tail -1 $O/smoke.log
timeout 900 python bench.py > $O/bench_ffn_8b.json 2> $O/bench_ffn_8b.err; tail -c 200 $O/bench_ffn_8b.json; echo
for w in attn lnmm ffn_70b lnmm_c1; do
  timeout 900 python bench.py --workload $w > $O/bench_$w.json 2> $O/bench_$w.err; tail -c 200 $O/bench_$w.json; echo
done
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_reference.json 2> $O/bench_reference.err; tail -c 200 $O/bench_reference.json; echo
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_bench_ffn.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-adapter > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_bench_attn.csv python bench.py --workload attn --steps 3 --warmup 3 --no-cpu-baseline --no-adapter > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ffn_swiglu -s 2 -c 1 -o $O/prof_ffn -f python scripts/ncu_target.py ffn_8b fused 3 > $O/ncu_ffn.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ln_matmul -s 2 -c 1 -o $O/prof_lnmm -f python scripts/ncu_target.py lnmm fused 3 > $O/ncu_lnmm.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_kernel -s 2 -c 1 -o $O/prof_attn -f python scripts/ncu_target.py attn fused 3 > $O/ncu_attn.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:f32 -s 4 -c 2 -o $O/prof_c1 -f python scripts/ncu_target.py lnmm_c1 fused 3 > $O/ncu_c1.log 2>&1
ls -la $O
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_f32x3 -s 1 -c 1 -o $O/prof_attn_f32 -f python scripts/ncu_fp32_target.py attn > $O/ncu_attn_f32.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"f32x3_(gemm|pair)" -s 2 -c 2 -o $O/prof_ffn_f32 -f python scripts/ncu_fp32_target.py ffn > $O/ncu_ffn_f32.log 2>&1
timeout 300 python scripts/fp32_modes.py > $O/fp32_modes.txt 2>&1
ls -la $O
