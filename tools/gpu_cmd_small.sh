mkdir -p gpurun_out
timeout 300 python tools/small_gemm_vs_cublas.py > gpurun_out/small_vs_cublas.json 2> gpurun_out/small_vs_cublas.err
M1='{"engine":1,"tile_m":128,"tile_n":64,"tile_k":64,"stages":8,"buffer_c":1,"acc_buffers":2,"persistent":1,"raster_group":4,"pack_warps":2}'
rm -f gpurun_out/trace_m1024.jsonl
XTC_TRACE=gpurun_out/trace_m1024.jsonl python tools/run_one.py matmul 1024 1024 1024 bf16 bf16 "$M1" 3 > /dev/null 2>&1
python tools/trace_report.py gpurun_out/trace_m1024.jsonl > gpurun_out/trace_m1024.txt 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_small.csv python tools/small_gemm_vs_cublas.py > /dev/null 2>&1
echo done
