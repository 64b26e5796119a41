# XTC_TRACE timelines of the small-GEMM bench schedules (512^3, 1024^3)
S512='{"engine":1,"tile_m":128,"tile_k":64,"swizzle":128,"tile_n":64,"stages":8,"buffer_c":1,"acc_buffers":1,"pack_warps":2}'
S1K='{"engine":1,"tile_m":128,"tile_k":64,"swizzle":128,"tile_n":64,"stages":8,"buffer_c":1,"acc_buffers":2,"persistent":1,"raster_group":4,"pack_warps":2}'
rm -f gpurun_out/trm*.jsonl
RUN_ONE_WARM=300 XTC_TRACE=gpurun_out/trm512.jsonl timeout 120 python tools/run_one.py matmul 512 512 512 bf16 bf16 "$S512" 1
RUN_ONE_WARM=300 XTC_TRACE=gpurun_out/trm1k.jsonl timeout 120 python tools/run_one.py matmul 1024 1024 1024 bf16 bf16 "$S1K" 1
