#!/bin/bash
# Functional test of bench.py's multi-rank path on one GPU: 2 ranks under torchrun (gloo, the
# ranks time-share the device). The numbers are not measurements; the JSON line is the check.
mkdir -p gpurun_out
for w in ffn_8b attn lnmm; do
  BFGPU_BENCH_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --workload $w --steps 5 --warmup 3 --sustained-s 0.5 --no-adapter > gpurun_out/mr_$w.json 2> gpurun_out/mr_$w.err
  echo "rc=$? $w"; tail -c 400 gpurun_out/mr_$w.json; echo; tail -3 gpurun_out/mr_$w.err
done
BFGPU_BENCH_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --impl reference --gpus 2 --steps 2 --warmup 1 > gpurun_out/mr_ref.json 2> gpurun_out/mr_ref.err
echo "rc=$? reference"; tail -c 300 gpurun_out/mr_ref.json
