#!/bin/bash
# Drop-in adapter with device-side transposes: parity (execute, CLI), adapter e2e at C3/C4/C5/C2/C1.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_execute.py tests/test_cli.py tests/test_abi.py tests/test_from_host_gpu.py -q -x -rf > gpurun_out/pytest_k.log 2>&1
tail -3 gpurun_out/pytest_k.log
nproc
for w in ffn_8b lnmm attn lnmm_c1 ffn_70b; do
  timeout 900 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_k_$w.json 2> gpurun_out/bench_k_$w.err
  python -c "import json; d=json.loads(open('gpurun_out/bench_k_$w.json').read().strip().splitlines()[-1]); a=d['e2e_adapter']; print('$w', round(d['value'],1), 'e2e', round(d['e2e']['value'],1), 'adapter', round(a.get('value',0),2), a.get('ms_per_call'), a.get('stages_ms_best_call'))"
done
