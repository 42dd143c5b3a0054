#!/bin/bash
./scripts/gpu_ab.sh base chunk -- --workload ffn_8b --steps 20 --warmup 5
./scripts/gpu_ab.sh base chunk -- --workload ffn_8b --rows 1024 --steps 20 --warmup 5
