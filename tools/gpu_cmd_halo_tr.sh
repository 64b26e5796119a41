mkdir -p gpurun_out
H='{"engine":1,"tile_m":128,"tile_n":64,"tile_k":64,"stages":2,"swizzle":128,"buffer_c":1,"acc_buffers":2,"persistent":1,"b_resident":1,"pack_halo":1}'
rm -f gpurun_out/trace_halo_m*.jsonl
for m in 0 7; do XTC_DEBUG_SKIP=$m XTC_TRACE=gpurun_out/trace_halo_m$m.jsonl timeout 120 python tools/run_one.py conv 32 56 56 64 64 bf16 bf16 "$H" 2 > /dev/null 2>&1; done
echo done
