L56='{"engine":1,"tile_m":128,"tile_k":64,"swizzle":128,"pack_halo":1,"buffer_c":1,"acc_buffers":2,"persistent":1,"tile_n":64,"stages":2,"b_resident":1}'
L56F='{"engine":1,"tile_m":128,"tile_k":64,"swizzle":128,"pack_halo":1,"buffer_c":1,"acc_buffers":2,"persistent":1,"tile_n":64,"stages":2,"b_resident":1,"inner_n":192}'
rm -f gpurun_out/tr*.jsonl
for sk in 7 1; do
XTC_DEBUG_SKIP=$sk RUN_ONE_WARM=300 XTC_TRACE=gpurun_out/tr56_s$sk.jsonl timeout 120 python tools/run_one.py conv 32 56 56 64 64 bf16 bf16 "$L56" 1
XTC_DEBUG_SKIP=$sk RUN_ONE_WARM=300 XTC_TRACE=gpurun_out/tr56f_s$sk.jsonl timeout 120 python tools/run_one.py conv 32 56 56 64 64 bf16 bf16 "$L56F" 1
done
./tools/umma_shift/timer_cost > gpurun_out/timer_cost.txt 2>&1
