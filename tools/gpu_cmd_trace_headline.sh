# XTC_TRACE of the 8192^3 headline schedule (pair 256x256x128, 3 stages): load latency and MMA stage gaps
mkdir -p gpurun_out; rm -f gpurun_out/trace_hl*.jsonl
H='{"engine":1,"tile_m":256,"tile_n":256,"tile_k":128,"stages":3,"swizzle":128,"buffer_c":1,"acc_buffers":2,"persistent":1,"raster_group":16,"order":0,"cluster_m":2}'
XTC_TRACE=gpurun_out/trace_hl.jsonl python tools/run_one.py matmul 8192 8192 8192 bf16 bf16 "$H" 20 > /dev/null 2>&1
python tools/trace_report.py gpurun_out/trace_hl.jsonl > gpurun_out/trace_hl.txt 2>&1
python -c "import sys; sys.path.insert(0,'tools'); import trace_report as t; t.grid_summary('gpurun_out/trace_hl.jsonl')" >> gpurun_out/trace_hl.txt 2>&1
echo done
