#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_attention_gpu.py tests/test_full_shape_gpu.py tests/test_snapshots_gpu.py tests/test_variants_gpu.py tests/test_concurrency_gpu.py -k "attention or attn or c2 or golden or shapes or extreme or snapshot or concurr" -q -x -rf > gpurun_out/pytest_attn.log 2>&1
tail -3 gpurun_out/pytest_attn.log
VARIANTS="old new nospec" bash scripts/gpu_ab_lib.sh --workload attn --steps 20 --warmup 5
