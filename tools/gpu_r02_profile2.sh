# round 2 (after the epilogue de-spill + LEAN variants): ncu --set full of the headline, conv L56 / L14 at N=32,
# 512^3 and the stem patch kernel; the bench launch list
H='{"engine":1,"tile_m":512,"tile_n":256,"tile_k":64,"stages":3,"swizzle":128,"buffer_c":1,"acc_buffers":1,"persistent":1,"raster_group":8,"order":0,"cluster_m":2}'
L56='{"engine":1,"tile_m":128,"tile_k":64,"swizzle":128,"pack_halo":1,"buffer_c":1,"acc_buffers":2,"persistent":1,"tile_n":64,"stages":2,"b_resident":1}'
L14='{"engine":1,"tile_m":256,"tile_k":128,"swizzle":128,"pack_halo":1,"buffer_c":1,"acc_buffers":2,"persistent":1,"cluster_m":2,"inner_m":256,"tile_n":128,"stages":3}'
S512='{"engine":1,"tile_m":128,"tile_k":64,"swizzle":128,"tile_n":64,"stages":8,"buffer_c":1,"acc_buffers":1,"pack_warps":2}'
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02b_launches.csv python bench.py --steps 5 --warmup 3 --no-extras --no-cpu-baseline > /dev/null 2>&1
timeout 400 ncu --set full --clock-control none --import-source on -k regex:tc_gemm -s 1 -c 1 -o gpurun_out/r02b_headline python tools/run_one.py matmul 8192 8192 8192 bf16 bf16 "$H" 2 > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:tc_conv_halo -s 1 -c 1 -o gpurun_out/r02b_conv56 python tools/run_one.py conv 32 56 56 64 64 bf16 bf16 "$L56" 2 > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:tc_conv_halo -s 1 -c 1 -o gpurun_out/r02b_conv14 python tools/run_one.py conv 32 14 14 256 256 bf16 bf16 "$L14" 2 > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:tc_gemm -s 1 -c 1 -o gpurun_out/r02b_mm512 python tools/run_one.py matmul 512 512 512 bf16 bf16 "$S512" 2 > /dev/null 2>&1
ls gpurun_out/*.ncu-rep
