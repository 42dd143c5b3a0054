#!/bin/bash
# Snapshot plans (staged K2/K3), 2-process shards, execute/CLI on every snapshot; staged bench lines.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_snapshots_gpu.py tests/test_sharded_gpu.py tests/test_cli.py tests/test_execute.py -q -x -rf > gpurun_out/pytest_i.log 2>&1
tail -15 gpurun_out/pytest_i.log
for w in attn lnmm; do
  for s in two_phase fused; do
    timeout 300 python bench.py --workload $w --schedule $s --steps 10 --warmup 3 --no-cpu-baseline --no-adapter > gpurun_out/bench_${w}_$s.json 2> gpurun_out/bench_${w}_$s.err
    python -c "import json; d=json.loads(open('gpurun_out/bench_${w}_$s.json').read().strip().splitlines()[-1]); print('$w $s', round(d['value'],1), round(d['ms_per_step'],4), d['gpu_launches'], d.get('check',{}).get('pass'))"
  done
done
