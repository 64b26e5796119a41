mkdir -p gpurun_out; rm -f gpurun_out/trace_wide*.jsonl
H='{"engine":1,"tile_m":512,"tile_n":256,"tile_k":64,"stages":4,"swizzle":128,"buffer_c":1,"acc_buffers":1,"persistent":1,"raster_group":8,"order":0,"cluster_m":2}'
XTC_TRACE=gpurun_out/trace_wide.jsonl python tools/run_one.py matmul 512 256 8192 bf16 bf16 "$H" 3 > /dev/null 2>&1
python tools/trace_report.py gpurun_out/trace_wide.jsonl > gpurun_out/trace_wide.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu.log
timeout 600 python tools/headline_epi_ab2.py > gpurun_out/headline_wide_ab.txt 2>&1
XTC_NO_WIDE_STORE=1 timeout 600 python tools/headline_epi_ab2.py > gpurun_out/headline_nowide_ab.txt 2>&1
timeout 600 python tools/headline_sustained_ab.py > gpurun_out/headline_sustained_ab5.txt 2>&1
echo done
