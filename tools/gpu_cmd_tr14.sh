mkdir -p gpurun_out
H='{"engine":1,"tile_m":128,"tile_n":128,"tile_k":128,"stages":3,"swizzle":128,"buffer_c":1,"acc_buffers":2,"persistent":1,"pack_halo":1}'
rm -f gpurun_out/trace_l14*.jsonl
for nb in 1 32; do XTC_TRACE=gpurun_out/trace_l14_n$nb.jsonl timeout 120 python tools/run_one.py conv $nb 14 14 256 256 bf16 bf16 "$H" 3 > /dev/null 2>&1; done
echo done
