mkdir -p gpurun_out; rm -f gpurun_out/trace4_*.jsonl
timeout 120 ./tools/tma_bench/tma_bench > gpurun_out/tma_bench.log 2>&1
C56='{"engine":1,"tile_m":128,"tile_n":64,"tile_k":64,"stages":8,"buffer_c":1,"acc_buffers":2,"persistent":1,"raster_group":8}'
P='{"engine":1,"tile_m":256,"tile_n":256,"tile_k":128,"stages":3,"buffer_c":1,"acc_buffers":2,"persistent":1,"raster_group":16,"cluster_m":2}'
XTC_TRACE=gpurun_out/trace4_c56.jsonl python tools/run_one.py conv 32 56 56 64 64 bf16 bf16 "$C56" 3 > /dev/null 2>&1
XTC_TRACE=gpurun_out/trace4_gemm_same.jsonl python tools/run_one.py matmul 100352 64 576 bf16 bf16 "$C56" 3 > /dev/null 2>&1
XTC_TRACE=gpurun_out/trace4_pair.jsonl python tools/run_one.py matmul 8192 8192 8192 bf16 bf16 "$P" 2 > /dev/null 2>&1
echo done
