#!/bin/bash
mkdir -p gpurun_out
for w in ffn_8b lnmm attn; do
  timeout 600 python bench.py --workload $w --no-cpu-baseline --no-adapter > gpurun_out/bench_sus_$w.json 2>gpurun_out/bench_sus_$w.err
  python -c "import json,sys; d=json.loads(open('gpurun_out/bench_sus_$w.json').read().strip().splitlines()[-1]); s=d['sustained']; print('$w', round(d['value'],1), 'sustained', round(s['value'],1), s['seconds'], s['frac_of_sustained_peak'], s['clocks'])"
done
