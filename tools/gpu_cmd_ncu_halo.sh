mkdir -p gpurun_out
H='{"engine":1,"tile_m":256,"tile_n":64,"tile_k":64,"stages":2,"swizzle":128,"buffer_c":1,"acc_buffers":2,"persistent":1,"b_resident":1,"pack_halo":1}'
I='{"engine":1,"tile_m":128,"tile_n":64,"tile_k":64,"stages":8,"swizzle":128,"buffer_c":1,"acc_buffers":2,"persistent":1,"raster_group":8,"pack_warps":3}'
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tc_conv_halo -s 1 -c 1 -o gpurun_out/ncu_halo_l56 -f python tools/run_one.py conv 32 56 56 64 64 bf16 bf16 "$H" 3 > gpurun_out/ncu_halo.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tc_gemm -s 1 -c 1 -o gpurun_out/ncu_im2col_l56 -f python tools/run_one.py conv 32 56 56 64 64 bf16 bf16 "$I" 3 >> gpurun_out/ncu_halo.log 2>&1
echo done
