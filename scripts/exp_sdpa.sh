timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv python scripts/ncu_sdpa.py 2>/dev/null | tail -8 > gpurun_out/sdpa_launches.csv
timeout 600 ncu --set full --clock-control none -k regex:"fmha|flash|sdpa|attention|cudnn" -s 1 -c 1 -o gpurun_out/prof_sdpa -f python scripts/ncu_sdpa.py > gpurun_out/ncu_sdpa.log 2>&1
tail -3 gpurun_out/ncu_sdpa.log
