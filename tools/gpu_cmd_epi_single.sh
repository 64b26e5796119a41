mkdir -p gpurun_out; rm -f gpurun_out/trace_single*.jsonl
H='{"engine":1,"tile_m":512,"tile_n":256,"tile_k":64,"stages":4,"swizzle":128,"buffer_c":1,"acc_buffers":1,"persistent":1,"raster_group":8,"order":0,"cluster_m":2}'
P='{"engine":1,"tile_m":256,"tile_n":256,"tile_k":128,"stages":3,"swizzle":128,"buffer_c":1,"acc_buffers":2,"persistent":1,"raster_group":16,"order":0,"cluster_m":2}'
XTC_TRACE=gpurun_out/trace_single.jsonl python tools/run_one.py matmul 512 256 8192 bf16 bf16 "$H" 3 > /dev/null 2>&1
XTC_TRACE=gpurun_out/trace_single_f32.jsonl python tools/run_one.py matmul 512 256 8192 bf16 f32 "$H" 3 > /dev/null 2>&1
XTC_TRACE=gpurun_out/trace_single256.jsonl python tools/run_one.py matmul 256 256 8192 bf16 bf16 "$P" 3 > /dev/null 2>&1
for f in trace_single trace_single_f32 trace_single256; do python tools/trace_report.py gpurun_out/$f.jsonl > gpurun_out/$f.txt 2>&1; done
echo done
