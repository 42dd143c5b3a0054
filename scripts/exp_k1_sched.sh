#!/bin/bash
# K1 fused vs two-phase at C3: per-launch ncu metrics (the two-phase step is two launches)
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors.sum,smsp__inst_executed.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second
echo "== fused"; timeout 300 ncu --metrics $M --clock-control none -k regex:ffn_swiglu -s 2 -c 1 --csv python scripts/ncu_target.py ffn_8b fused 3 2>/dev/null | grep -E '"(gpu__|smsp__|sm__|lts__|dram__)' | awk -F'","' '{print $(NF-2), $NF}'
echo "== two_phase (gate/up, down)"; timeout 300 ncu --metrics $M --clock-control none -k regex:ffn_swiglu -s 4 -c 2 --csv python scripts/ncu_target.py ffn_8b two_phase 3 2>/dev/null | grep -E '"(gpu__|smsp__|sm__|lts__|dram__)' | awk -F'","' '{print $(NF-2), $NF}'
