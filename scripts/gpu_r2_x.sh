#!/bin/bash
# K1 split down tiles: parity, then unsplit (BFGPU_FFN_KSPLIT=1) vs split at the shard sizes and full C3.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_ffn_gpu.py tests/test_full_shape_gpu.py tests/test_variants_gpu.py tests/test_sharded_gpu.py tests/test_from_host_gpu.py tests/test_concurrency_gpu.py -q -x -rf -k "ffn or c3 or c5 or ragged or shard or host or concurr or K1 or variant" > gpurun_out/pytest_ksplit.log 2>&1
tail -4 gpurun_out/pytest_ksplit.log
for rows in 1024 2048 4096 8192; do
  for rep in 1 2; do
    for ks in 1 2; do
      r=$(BFGPU_FFN_KSPLIT=$ks timeout 300 python bench.py --rows $rows --steps 20 --warmup 5 --no-cpu-baseline --no-adapter --no-check 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['value'],1), round(d['ms_per_step'],4), d['clocks']['sm_mhz'], d['plan']['ksplit'], round(d['plan']['sched_eff'],3))")
      echo "rows=$rows ks=$ks $r"
    done
  done
done
