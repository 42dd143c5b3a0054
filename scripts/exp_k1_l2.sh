#!/bin/bash
cp paper_2505_07829_b200/lib/libbfgpu.so /tmp/libbfgpu_base.so
for v in base hint; do
  if [ $v = hint ]; then cp variants/libbfgpu_hint.so paper_2505_07829_b200/lib/libbfgpu.so; else cp /tmp/libbfgpu_base.so paper_2505_07829_b200/lib/libbfgpu.so; fi
  echo "$v: $(timeout 120 python scripts/quick_perf.py ffn 2>&1 | grep fused)"
  timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:ffn_swiglu -s 2 -c 1 --csv python scripts/ncu_target.py ffn_8b fused 3 2>/dev/null | grep -E 'dram__bytes' | awk -F'","' '{print $(NF-2), $(NF-1), $NF}'
done
cp /tmp/libbfgpu_base.so paper_2505_07829_b200/lib/libbfgpu.so
