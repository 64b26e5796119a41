mkdir -p gpurun_out; rm -f gpurun_out/trace3_*.jsonl
C56='{"engine":1,"tile_m":128,"tile_n":64,"tile_k":64,"stages":8,"buffer_c":1,"acc_buffers":2,"persistent":1,"raster_group":8}'
P='{"engine":1,"tile_m":256,"tile_n":256,"tile_k":128,"stages":3,"buffer_c":1,"acc_buffers":2,"persistent":1,"raster_group":16,"cluster_m":2}'
M1='{"engine":1,"tile_m":128,"tile_n":64,"tile_k":64,"stages":8,"buffer_c":1,"acc_buffers":2,"persistent":1,"raster_group":4}'
XTC_TRACE=gpurun_out/trace3_c56.jsonl python tools/run_one.py conv 32 56 56 64 64 bf16 bf16 "$C56" 3 > /dev/null 2>&1
XTC_TRACE=gpurun_out/trace3_gemm_same.jsonl python tools/run_one.py matmul 100352 64 576 bf16 bf16 "$C56" 3 > /dev/null 2>&1
XTC_TRACE=gpurun_out/trace3_pair.jsonl python tools/run_one.py matmul 8192 8192 8192 bf16 bf16 "$P" 2 > /dev/null 2>&1
XTC_TRACE=gpurun_out/trace3_m1024.jsonl python tools/run_one.py matmul 1024 1024 1024 bf16 bf16 "$M1" 3 > /dev/null 2>&1
timeout 300 python tools/conv_diag.py > gpurun_out/conv_diag2.log 2>&1
timeout 300 python tools/quick_perf4.py > gpurun_out/quick_perf4b.log 2>&1
timeout 600 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 300 > gpurun_out/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu.log
echo done
