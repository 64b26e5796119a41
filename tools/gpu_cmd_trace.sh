mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 300 -x > gpurun_out/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu.log
C56='{"engine":1,"tile_m":128,"tile_n":64,"tile_k":64,"stages":8,"buffer_c":1,"acc_buffers":2,"persistent":1,"raster_group":8}'
C56b='{"engine":1,"tile_m":128,"tile_n":64,"tile_k":64,"stages":6,"buffer_c":1,"acc_buffers":2,"persistent":0}'
P='{"engine":1,"tile_m":256,"tile_n":256,"tile_k":128,"stages":3,"buffer_c":1,"acc_buffers":2,"persistent":1,"raster_group":16,"cluster_m":2}'
M1='{"engine":1,"tile_m":128,"tile_n":64,"tile_k":64,"stages":8,"buffer_c":1,"acc_buffers":2,"persistent":1,"raster_group":4}'
rm -f gpurun_out/trace_*.jsonl
XTC_TRACE=gpurun_out/trace_c56.jsonl python tools/run_one.py conv 32 56 56 64 64 bf16 bf16 "$C56" 3 > /dev/null 2>&1
XTC_TRACE=gpurun_out/trace_c56np.jsonl python tools/run_one.py conv 32 56 56 64 64 bf16 bf16 "$C56b" 3 > /dev/null 2>&1
XTC_TRACE=gpurun_out/trace_pair.jsonl python tools/run_one.py matmul 8192 8192 8192 bf16 bf16 "$P" 3 > /dev/null 2>&1
XTC_TRACE=gpurun_out/trace_m1024.jsonl python tools/run_one.py matmul 1024 1024 1024 bf16 bf16 "$M1" 3 > /dev/null 2>&1
timeout 300 python tools/simt_probe.py > gpurun_out/simt_probe.log 2>&1
echo done
