timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv python scripts/ncu_cublas.py 2>/dev/null | grep -v "randn\|copy\|distribution" | tail -3 > gpurun_out/cublas_launches.csv
timeout 600 ncu --set full --clock-control none -k regex:"gemm|sm100|nvjet|cutlass" -s 1 -c 1 -o gpurun_out/prof_cublas -f python scripts/ncu_cublas.py > gpurun_out/ncu_cublas.log 2>&1
tail -2 gpurun_out/ncu_cublas.log
