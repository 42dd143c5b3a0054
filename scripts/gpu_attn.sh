timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -1 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 300 python bench.py --workload attn --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_attn.json 2> gpurun_out/bench_attn.err; tail -c 300 gpurun_out/bench_attn.json
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_kernel -s 2 -c 1 -o gpurun_out/prof_attn -f python scripts/ncu_target.py attn fused 3 > gpurun_out/ncu_attn.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_attn.csv python bench.py --workload attn --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_attn_under_ncu.log 2>&1
