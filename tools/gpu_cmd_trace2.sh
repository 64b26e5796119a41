mkdir -p gpurun_out; rm -f gpurun_out/trace2_*.jsonl
C56='{"engine":1,"tile_m":128,"tile_n":64,"tile_k":64,"stages":8,"buffer_c":1,"acc_buffers":2,"persistent":1,"raster_group":8}'
C56s4='{"engine":1,"tile_m":128,"tile_n":64,"tile_k":64,"stages":4,"buffer_c":1,"acc_buffers":2,"persistent":1,"raster_group":8}'
G128='{"engine":1,"tile_m":128,"tile_n":128,"tile_k":64,"stages":6,"buffer_c":1,"acc_buffers":2,"persistent":1,"raster_group":8}'
XTC_TRACE=gpurun_out/trace2_gemm_same.jsonl python tools/run_one.py matmul 100352 64 576 bf16 bf16 "$C56" 3 > /dev/null 2>&1
XTC_TRACE=gpurun_out/trace2_c56s4.jsonl python tools/run_one.py conv 32 56 56 64 64 bf16 bf16 "$C56s4" 3 > /dev/null 2>&1
XTC_TRACE=gpurun_out/trace2_c56n128.jsonl python tools/run_one.py conv 32 56 56 64 128 bf16 bf16 "$G128" 3 > /dev/null 2>&1
XTC_TRACE=gpurun_out/trace2_c14.jsonl python tools/run_one.py conv 32 14 14 256 256 bf16 bf16 '{"engine":1,"tile_m":128,"tile_n":256,"tile_k":64,"stages":4,"buffer_c":1,"acc_buffers":2,"persistent":1}' 3 > /dev/null 2>&1
XTC_TRACE=gpurun_out/trace2_gemm8k_1cta.jsonl python tools/run_one.py matmul 8192 8192 8192 bf16 bf16 '{"engine":1,"tile_m":128,"tile_n":256,"tile_k":64,"stages":4,"buffer_c":1,"acc_buffers":2,"persistent":1,"raster_group":16}' 2 > /dev/null 2>&1
echo done
