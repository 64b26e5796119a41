mkdir -p gpurun_out
H='{"engine":1,"tile_m":256,"tile_n":64,"tile_k":64,"stages":2,"swizzle":128,"buffer_c":1,"acc_buffers":2,"persistent":1,"b_resident":1,"pack_halo":1}'
timeout 300 python tools/halo_diag.py "$H" > gpurun_out/halo_diag.log 2>&1
for m in 1 2 4; do XTC_DEBUG_SKIP=$m XTC_TRACE=gpurun_out/trace_halo_m$m.jsonl timeout 120 python tools/run_one.py conv 32 56 56 64 64 bf16 bf16 "$H" 2 >> gpurun_out/halo_diag.log 2>&1; done
echo done
