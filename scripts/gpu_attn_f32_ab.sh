#!/bin/bash
# K3 fp32 A/B of two library builds on one box (variants/libbfgpu_{attnold,attnnew}.so)
L=paper_2505_07829_b200/lib/libbfgpu.so
cp $L /tmp/libbfgpu_intree.so
for rep in 1 2 3; do
  for v in attnold attnnew; do
    cp variants/libbfgpu_$v.so $L
    echo "$v $(python scripts/fp32_modes.py 2>&1 | sed -n 5p)"
  done
done
cp /tmp/libbfgpu_intree.so $L
