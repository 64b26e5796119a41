L56='{"engine":1,"tile_m":128,"tile_k":64,"swizzle":128,"pack_halo":2,"buffer_c":0,"acc_buffers":2,"persistent":1,"tile_n":64,"stages":2,"b_resident":1}'
timeout 600 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "halo or conv" > gpurun_out/t_halo.log 2>&1
PYTHONPATH=. timeout 300 python tools/ab_mean.py conv 32 56 64 cudnn "env=0:$L56" "env=32768:$L56" > gpurun_out/ab_tap9.txt 2>&1
PYTHONPATH=. timeout 300 python tools/ab_mean.py conv 8 56 64 cudnn "env=0:$L56" "env=32768:$L56" >> gpurun_out/ab_tap9.txt 2>&1
RUN_ONE_WARM=300 XTC_TRACE=gpurun_out/tr56t9.jsonl timeout 120 python tools/run_one.py conv 32 56 56 64 64 bf16 bf16 "$L56" 1 > /dev/null 2>&1
python tools/trace_report.py gpurun_out/tr56t9.jsonl > gpurun_out/tr56t9.rep.txt 2>&1
python tools/trace_phases.py gpurun_out/tr56t9.jsonl > gpurun_out/tr56t9.ph.txt 2>&1
