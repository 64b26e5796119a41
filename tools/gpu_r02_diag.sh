P='{"engine":1,"tile_m":256,"cluster_m":2,"inner_m":256,"tile_k":64,"swizzle":128,"pack_halo":1,"acc_buffers":2,"persistent":1,"tile_n":64,"stages":2,"b_resident":1,"buffer_c":0}'
RUN_ONE_WARM=300 XTC_TRACE=gpurun_out/tr56p64.jsonl timeout 120 python tools/run_one.py conv 32 56 56 64 64 bf16 bf16 "$P" 1 > /dev/null 2>&1
python tools/trace_report.py gpurun_out/tr56p64.jsonl > gpurun_out/tr56p64.rep.txt 2>&1
python tools/trace_phases.py gpurun_out/tr56p64.jsonl > gpurun_out/tr56p64.ph.txt 2>&1
