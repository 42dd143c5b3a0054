#!/bin/bash
# A/B of two builds of libbfgpu.so on one box: scripts/gpu_ab.sh <variantA> <variantB> -- <bench args...>
# Each variant runs alternately, three times.
mkdir -p gpurun_out
A=$1; B=$2; shift 3
for rep in 1 2 3; do
  for v in $A $B; do
    cp variants/libbfgpu_$v.so paper_2505_07829_b200/lib/libbfgpu.so
    r=$(timeout 300 python bench.py "$@" --no-cpu-baseline --no-adapter --no-check 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['value'],1), round(d['ms_per_step'],4), d['clocks']['sm_mhz'])")
    echo "$v $* : $r"
  done
done
