mkdir -p gpurun_out; rm -f gpurun_out/trace_ovl*.jsonl
H='{"engine":1,"tile_m":512,"tile_n":256,"tile_k":64,"stages":3,"swizzle":128,"buffer_c":1,"acc_buffers":1,"persistent":1,"raster_group":8,"order":0,"cluster_m":2}'
timeout 900 python -m pytest tests -m gpu -x -q -k "subtiles or overlapped or gather" > gpurun_out/pytest_ovl.log 2>&1; echo rc=$? >> gpurun_out/pytest_ovl.log
XTC_TRACE=gpurun_out/trace_ovl.jsonl python tools/run_one.py matmul 8192 8192 8192 bf16 bf16 "$H" 3 > /dev/null 2>&1
python tools/trace_report.py gpurun_out/trace_ovl.jsonl > gpurun_out/trace_ovl.txt 2>&1
timeout 600 python tools/headline_ovl_ab.py > gpurun_out/headline_ovl_ab.txt 2>&1
XTC_NO_OVERLAP_EPILOGUE=1 timeout 600 python tools/headline_ovl_ab.py > gpurun_out/headline_noovl_ab.txt 2>&1
echo done
