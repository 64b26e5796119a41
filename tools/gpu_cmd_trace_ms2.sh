mkdir -p gpurun_out; rm -f gpurun_out/trace_ms2.jsonl
H='{"engine":1,"tile_m":512,"tile_n":256,"tile_k":64,"stages":4,"swizzle":128,"buffer_c":1,"acc_buffers":1,"persistent":1,"raster_group":8,"order":0,"cluster_m":2}'
XTC_TRACE=gpurun_out/trace_ms2.jsonl python tools/run_one.py matmul 8192 8192 8192 bf16 bf16 "$H" 3 > /dev/null 2>&1
python tools/trace_report.py gpurun_out/trace_ms2.jsonl > gpurun_out/trace_ms2.txt 2>&1
echo done
