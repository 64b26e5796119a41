mkdir -p gpurun_out
M1='{"engine":1,"tile_m":128,"tile_n":64,"tile_k":64,"stages":4,"buffer_c":1,"acc_buffers":2,"persistent":0,"raster_group":8,"tile_k":128}'
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_small.csv python tools/small_gemm_vs_cublas.py > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none -k regex:"(gemm|nvjet|cutlass|sm100|Kernel)" -s 1 -c 1 -o gpurun_out/prof_cublas1024 -f python tools/cublas_small_one.py 1024 > gpurun_out/ncu_cublas1024.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:tc_gemm -s 1 -c 1 -o gpurun_out/prof_xtc1024 -f python tools/run_one.py matmul 1024 1024 1024 bf16 bf16 "$M1" 3 > gpurun_out/ncu_xtc1024.log 2>&1
echo done
