#!/bin/bash
# K1 k-step sync: parity with it forced on, then C5 DRAM and throughput per setting.
mkdir -p gpurun_out
BFGPU_FFN_KSYNC=8 timeout 900 python -m pytest tests/test_ffn_gpu.py tests/test_full_shape_gpu.py -q -x -rf -k "ffn or c3 or c5 or ragged" > gpurun_out/pytest_ks.log 2>&1
tail -2 gpurun_out/pytest_ks.log
M="dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second"
for cfg in "BFGPU_FFN_KSYNC=0" "BFGPU_FFN_KSYNC=16" "BFGPU_FFN_KSYNC=8" "BFGPU_FFN_KSYNC=16 BFGPU_FFN_KSLACK=4" "BFGPU_FFN_KSYNC=16 BFGPU_FFN_WAVESYNC=0"; do
  echo "== $cfg"
  env $cfg timeout 300 ncu --metrics $M --clock-control none -k regex:ffn_swiglu -s 1 -c 1 --csv python scripts/ncu_target.py ffn_70b fused 2 2>/dev/null | grep -E 'dram__bytes|gpu__time|tensor|per_second' | awk -F'","' '{print $(NF-2), $(NF-1), $NF}'
  env $cfg timeout 300 python bench.py --workload ffn_70b --steps 10 --warmup 3 --no-cpu-baseline --no-adapter --no-check 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('bench', round(d['value'],1), round(d['ms_per_step'],3))"
done
