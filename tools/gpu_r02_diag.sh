P='"engine":1,"swizzle":128,"pack_halo":1,"acc_buffers":2,"persistent":1,"tile_m":256,"cluster_m":2,"inner_m":256,"tile_k":128,"tile_n":128,"stages":3'
for bc in 0 1; do
RUN_ONE_WARM=100 XTC_TRACE=gpurun_out/tr14p$bc.jsonl timeout 120 python tools/run_one.py conv 32 14 14 256 256 bf16 bf16 "{$P,\"buffer_c\":$bc}" 1 > /dev/null 2>&1
python tools/trace_report.py gpurun_out/tr14p$bc.jsonl > gpurun_out/tr14p$bc.rep.txt 2>&1
python tools/trace_phases.py gpurun_out/tr14p$bc.jsonl > gpurun_out/tr14p$bc.ph.txt 2>&1
done
