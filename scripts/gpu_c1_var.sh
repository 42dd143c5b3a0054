#!/bin/bash
# C1 warm per-call time for library variants (VARIANTS="base noepi ..." bash scripts/gpu_c1_var.sh)
L=paper_2505_07829_b200/lib/libbfgpu.so
cp $L /tmp/libbfgpu_intree.so
for rep in 1 2; do
  for v in ${VARIANTS:-base}; do
    cp variants/libbfgpu_$v.so $L
    echo "$v $(timeout 120 python scripts/c1_breakdown.py 2>&1 | tail -1)"
  done
done
cp /tmp/libbfgpu_intree.so $L
