#!/bin/bash
# A/B builds of libbfgpu.so on one box: VARIANTS="old new" bash scripts/gpu_ab_lib.sh <bench args...>
# (variants/libbfgpu_<name>.so, built by scripts/build_variant.sh); the in-tree build is restored at the end.
mkdir -p gpurun_out
L=paper_2505_07829_b200/lib/libbfgpu.so
cp $L /tmp/libbfgpu_intree.so
for rep in 1 2 3; do
  for v in ${VARIANTS:-old new}; do
    cp variants/libbfgpu_$v.so $L
    r=$(timeout 300 python bench.py "$@" --no-cpu-baseline --no-adapter --no-check 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['value'],1), round(d['ms_per_step'],4))")
    echo "$v $r"
  done
done
cp /tmp/libbfgpu_intree.so $L
