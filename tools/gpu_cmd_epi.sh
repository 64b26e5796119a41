mkdir -p gpurun_out
P='{"engine":1,"tile_m":512,"tile_n":256,"tile_k":64,"stages":4,"swizzle":128,"buffer_c":1,"acc_buffers":1,"persistent":1,"raster_group":8,"order":0,"cluster_m":2}'
A='{"engine":1,"tile_m":128,"tile_n":64,"tile_k":64,"stages":8,"buffer_c":1,"swizzle":128}'
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu.log
rm -f gpurun_out/trace_epi.jsonl
XTC_TRACE=gpurun_out/trace_epi.jsonl python tools/run_one.py matmul 1024 1024 1024 bf16 bf16 "$A" 3 > /dev/null 2>&1
python tools/trace_report.py gpurun_out/trace_epi.jsonl > gpurun_out/trace_epi.txt 2>&1
timeout 600 python tools/headline_sustained_ab.py > gpurun_out/headline_sustained_ab2.txt 2>&1
timeout 600 python tools/headline_msub_ab2.py > gpurun_out/headline_msub_ab3.txt 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:tc_gemm -s 1 -c 1 -o gpurun_out/prof_headline_final5 -f python tools/run_one.py matmul 8192 8192 8192 bf16 bf16 "$P" 2 > gpurun_out/ncu_final5.log 2>&1
timeout 300 python tools/small_gemm_vs_cublas.py > gpurun_out/small_vs_cublas3.json 2> gpurun_out/small_vs_cublas3.err
echo done
