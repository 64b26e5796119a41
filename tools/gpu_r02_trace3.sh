# XTC_TRACE timelines of the bench's conv schedules (L56 / L14 at N=32), flushed-L2 single launches after warm-up
L56='{"engine":1,"tile_m":128,"tile_k":64,"swizzle":128,"pack_halo":1,"buffer_c":1,"acc_buffers":2,"persistent":1,"tile_n":64,"stages":2,"b_resident":1}'
L14='{"engine":1,"tile_m":128,"tile_k":128,"swizzle":128,"pack_halo":1,"buffer_c":1,"acc_buffers":2,"persistent":1,"tile_n":128,"stages":3}'
rm -f gpurun_out/tr*.jsonl
RUN_ONE_WARM=300 XTC_TRACE=gpurun_out/tr56.jsonl timeout 120 python tools/run_one.py conv 32 56 56 64 64 bf16 bf16 "$L56" 1 > gpurun_out/tr.log 2>&1
RUN_ONE_WARM=300 XTC_TRACE=gpurun_out/tr14.jsonl timeout 120 python tools/run_one.py conv 32 14 14 256 256 bf16 bf16 "$L14" 1 >> gpurun_out/tr.log 2>&1
for f in tr56 tr14; do
 python tools/trace_report.py gpurun_out/$f.jsonl grid > gpurun_out/$f.grid.txt 2>&1
 python tools/trace_report.py gpurun_out/$f.jsonl > gpurun_out/$f.rep.txt 2>&1
 python tools/trace_phases.py gpurun_out/$f.jsonl > gpurun_out/$f.ph.txt 2>&1
done
python tools/cudnn_conv_ref.py > gpurun_out/cudnn.txt 2>&1
