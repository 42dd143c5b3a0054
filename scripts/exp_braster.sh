#!/bin/bash
timeout 600 python -m pytest tests/test_ffn_gpu.py -x -q 2>&1 | tail -1
BFGPU_FFN_BRASTER=8 timeout 600 python -m pytest tests/test_ffn_gpu.py -x -q 2>&1 | tail -1
BFGPU_FFN_BRASTER=2 timeout 600 python -m pytest tests/test_ffn_gpu.py -x -q 2>&1 | tail -1
M=gpu__time_duration.sum,dram__bytes_read.sum,sm__cycles_elapsed.avg.per_second
for br in 0 8 4; do for sch in fused two_phase; do echo "braster $br $sch"; BFGPU_FFN_BRASTER=$br timeout 300 ncu --metrics $M --clock-control none -k regex:ffn_swiglu -s 2 -c 2 --csv python scripts/ncu_target.py ffn_8b $sch 3 2>/dev/null | grep -E '"(gpu__|sm__|dram__)' | awk -F'","' '{print $(NF-2), $NF}'; done; done
for r in 1 2; do for br in 0 8; do BFGPU_FFN_BRASTER=$br timeout 300 python scripts/exp_power.py ffn 2>&1 | tail -1 | sed "s/^/braster $br: /"; done; done
