#!/bin/bash
# fp32 C1 kernel check + the 8-GPU shard sizes on one GPU (strong-scaling prediction)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "fp32 or f32 or c1 or codegen" > gpurun_out/pytest_e.log 2>&1
timeout 600 python bench.py --workload lnmm_c1 --steps 50 --warmup 5 --no-cpu-baseline --no-adapter > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_f32 -s 2 -c 1 -o gpurun_out/prof_c1 -f python scripts/ncu_target.py lnmm_c1 fused 3 > gpurun_out/ncu_c1.log 2>&1
for spec in "ffn_8b 1024" "ffn_8b 2048" "ffn_8b 4096" "ffn_70b 4096" "ffn_70b 8192" "lnmm 8192" "attn 32"; do
  set -- $spec
  timeout 600 python bench.py --workload $1 --rows $2 --steps 20 --warmup 5 --no-cpu-baseline --no-adapter > gpurun_out/shard_$1_$2.json 2> gpurun_out/shard_$1_$2.err
done
for w in ffn_8b ffn_70b lnmm attn; do
  timeout 600 python bench.py --workload $w --steps 20 --warmup 5 --no-cpu-baseline --no-adapter > gpurun_out/full_$w.json 2> gpurun_out/full_$w.err
done
tail -3 gpurun_out/pytest_e.log
