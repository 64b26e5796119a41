# XTC_TRACE timelines of the BASELINE conv layers at N=32 (+ XTC_DEBUG_SKIP decompositions for L56)
L14='{"engine":1,"tile_m":256,"tile_k":128,"swizzle":128,"pack_halo":1,"buffer_c":1,"acc_buffers":2,"persistent":1,"cluster_m":2,"inner_m":256,"tile_n":128,"stages":3}'
L56='{"engine":1,"tile_m":128,"tile_k":64,"swizzle":128,"pack_halo":1,"buffer_c":1,"acc_buffers":2,"persistent":1,"tile_n":64,"stages":2,"b_resident":1}'
rm -f gpurun_out/tr*.jsonl
XTC_TRACE=gpurun_out/tr14.jsonl timeout 120 python tools/run_one.py conv 32 14 14 256 256 bf16 bf16 "$L14" 3
XTC_TRACE=gpurun_out/tr56.jsonl timeout 120 python tools/run_one.py conv 32 56 56 64 64 bf16 bf16 "$L56" 3
for sk in 1 2 4 6; do
XTC_DEBUG_SKIP=$sk XTC_TRACE=gpurun_out/tr56_skip$sk.jsonl timeout 120 python tools/run_one.py conv 32 56 56 64 64 bf16 bf16 "$L56" 3
done
