#!/bin/bash
cp paper_2505_07829_b200/lib/libbfgpu.so /tmp/libbfgpu_R2.so
for R in 1 2 4 8; do
  if [ $R != 2 ]; then cp variants/libbfgpu_R$R.so paper_2505_07829_b200/lib/libbfgpu.so; else cp /tmp/libbfgpu_R2.so paper_2505_07829_b200/lib/libbfgpu.so; fi
  echo "rows=$R: $(timeout 120 python scripts/quick_perf.py lnmm 2>&1 | grep 'K2:')  $(timeout 120 python scripts/quick_perf.py lnmm 2>&1 | grep 'K2:')"
done
cp /tmp/libbfgpu_R2.so paper_2505_07829_b200/lib/libbfgpu.so
