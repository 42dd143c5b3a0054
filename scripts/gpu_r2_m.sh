#!/bin/bash
mkdir -p gpurun_out
timeout 3000 python scripts/snapshot_traffic.py > gpurun_out/snapshot_traffic.log 2>&1
tail -30 gpurun_out/snapshot_traffic.log
