#!/bin/bash
# C5 DRAM breakdown: per-launch DRAM bytes, L2 hit rate and time for the two-phase and fused
# schedules under a few scheduling groups / down rasters.
mkdir -p gpurun_out
M="dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct,lts__t_sectors_srcunit_tex.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second"
run() {
  echo "== $*"
  env "$@" timeout 300 ncu --metrics $M --clock-control none -k regex:ffn_swiglu -s 2 -c 2 --csv python scripts/ncu_target.py ffn_70b $SCHED 2 2>/dev/null | grep -E 'dram__bytes|gpu__time|hit_rate|srcunit_tex|tensor|per_second' | awk -F'","' '{print $(NF-3), $(NF-2), $(NF-1), $NF}'
}
SCHED=two_phase run BFGPU_NOP=1
SCHED=two_phase run BFGPU_FFN_GROUP=8
SCHED=two_phase run BFGPU_FFN_GROUP=32
SCHED=two_phase run BFGPU_FFN_BRASTER=2
SCHED=fused run BFGPU_NOP=1
SCHED=fused run BFGPU_FFN_BRASTER=2
