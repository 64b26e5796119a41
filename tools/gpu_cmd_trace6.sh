mkdir -p gpurun_out; rm -f gpurun_out/trace6_*.jsonl
C56='{"engine":1,"tile_m":128,"tile_n":64,"tile_k":64,"stages":7,"buffer_c":1,"acc_buffers":2,"persistent":1,"raster_group":8,"pack_warps":3,"b_resident":1}'
XTC_TRACE=gpurun_out/trace6_c56.jsonl python tools/run_one.py conv 32 56 56 64 64 bf16 bf16 "$C56" 2 > /dev/null 2>&1
C14='{"engine":1,"tile_m":256,"cluster_m":2,"tile_n":256,"tile_k":128,"stages":3,"buffer_c":1,"acc_buffers":2,"persistent":1,"pack_warps":2}'
XTC_TRACE=gpurun_out/trace6_c14.jsonl python tools/run_one.py conv 32 14 14 256 256 bf16 bf16 "$C14" 2 > /dev/null 2>&1
M1='{"engine":1,"tile_m":128,"tile_n":64,"tile_k":64,"stages":8,"buffer_c":1,"acc_buffers":2,"persistent":1,"raster_group":4,"pack_warps":2}'
XTC_TRACE=gpurun_out/trace6_m1024.jsonl python tools/run_one.py matmul 1024 1024 1024 bf16 bf16 "$M1" 2 > /dev/null 2>&1
echo done
