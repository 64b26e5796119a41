mkdir -p gpurun_out; rm -f gpurun_out/trace7_*.jsonl
C56='{"engine":1,"tile_m":128,"tile_n":64,"tile_k":64,"stages":8,"buffer_c":1,"acc_buffers":2,"persistent":1,"raster_group":8,"pack_warps":3}'
XTC_TRACE=gpurun_out/trace7_c56.jsonl python tools/run_one.py conv 32 56 56 64 64 bf16 bf16 "$C56" 2 > /dev/null 2>&1
XTC_DEBUG_SKIP_MMA=1 XTC_TRACE=gpurun_out/trace7_c56_skip.jsonl python tools/run_one.py conv 32 56 56 64 64 bf16 bf16 "$C56" 2 > /dev/null 2>&1
timeout 300 python tools/simt_probe.py > gpurun_out/simt_probe3.log 2>&1
echo done
