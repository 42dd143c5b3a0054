#!/bin/bash
# K2 512x256 tiles (BFGPU_LNMM_WIDE=1): parity, then A/B burst and sustained against 256x256.
mkdir -p gpurun_out
BFGPU_LNMM_WIDE=1 timeout 900 python -m pytest tests -m gpu -q -x -rf -k "lnmm or layernorm or c4 or c1 or K2 or concurr or shard" > gpurun_out/pytest_wide.log 2>&1
tail -3 gpurun_out/pytest_wide.log
for rep in 1 2 3; do
  for w in 0 1; do
    r=$(BFGPU_LNMM_WIDE=$w timeout 300 python bench.py --workload lnmm --steps 20 --warmup 5 --no-cpu-baseline --no-adapter --no-check 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); s=d['sustained']; print(round(d['value'],1), round(d['ms_per_step'],4), 'sustained', round(s['value'],1), s['clocks']['sm_mhz'], d['plan']['kernel'])")
    echo "wide=$w $r"
  done
done
BFGPU_LNMM_WIDE=1 timeout 300 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second,l1tex__m_xbar2l1tex_read_bytes.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:ln_matmul -s 2 -c 1 --csv python scripts/ncu_target.py lnmm fused 3 2>/dev/null | grep -E 'gpu__time|tensor|per_second|xbar|dram' | awk -F'","' '{print $(NF-2), $(NF-1), $NF}'
