mkdir -p gpurun_out; rm -f gpurun_out/trace5_*.jsonl
C56='{"engine":1,"tile_m":128,"tile_n":64,"tile_k":64,"stages":8,"buffer_c":1,"acc_buffers":2,"persistent":1,"raster_group":8,"pack_warps":3}'
XTC_TRACE=gpurun_out/trace5_c56.jsonl python tools/run_one.py conv 32 56 56 64 64 bf16 bf16 "$C56" 3 > /dev/null 2>&1
M1='{"engine":1,"tile_m":128,"tile_n":64,"tile_k":64,"stages":8,"buffer_c":1,"acc_buffers":2,"persistent":1,"raster_group":4,"pack_warps":2}'
XTC_TRACE=gpurun_out/trace5_m1024.jsonl python tools/run_one.py matmul 1024 1024 1024 bf16 bf16 "$M1" 3 > /dev/null 2>&1
timeout 400 python tools/quick_perf5.py > gpurun_out/quick_perf5b.log 2>&1
echo done
