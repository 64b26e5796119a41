T='"engine":1,"tile_m":128,"swizzle":128,"buffer_c":1'
PYTHONPATH=. timeout 250 python tools/ab_mean.py matmul 512 cublas \
 "{$T,\"tile_k\":128,\"tile_n\":64,\"stages\":4,\"acc_buffers\":1,\"pack_warps\":2}" \
 "{$T,\"tile_k\":64,\"tile_n\":64,\"stages\":4,\"acc_buffers\":1,\"split_k\":2,\"split_k_mode\":2,\"buffer_c\":0}" \
 "{$T,\"tile_k\":64,\"tile_n\":64,\"stages\":2,\"acc_buffers\":1,\"split_k\":4,\"split_k_mode\":2,\"buffer_c\":0}" \
 "{$T,\"tile_k\":64,\"tile_n\":128,\"stages\":2,\"acc_buffers\":1,\"split_k\":4,\"split_k_mode\":2,\"buffer_c\":0}" \
 "{$T,\"tile_k\":64,\"tile_n\":64,\"stages\":4,\"acc_buffers\":2,\"persistent\":1,\"split_k_mode\":3}" > gpurun_out/ab_small.txt 2>&1
PYTHONPATH=. timeout 250 python tools/ab_mean.py matmul 1024 cublas \
 "{$T,\"tile_k\":128,\"tile_n\":64,\"stages\":3,\"acc_buffers\":2,\"persistent\":0,\"raster_group\":2}" \
 "{$T,\"tile_k\":64,\"tile_n\":128,\"stages\":4,\"acc_buffers\":1,\"split_k\":2,\"split_k_mode\":2,\"buffer_c\":0}" \
 "{$T,\"tile_k\":64,\"tile_n\":64,\"stages\":4,\"acc_buffers\":1,\"split_k\":2,\"split_k_mode\":2,\"buffer_c\":0}" \
 "{$T,\"tile_k\":64,\"tile_n\":128,\"stages\":4,\"acc_buffers\":2,\"persistent\":1,\"split_k_mode\":3}" >> gpurun_out/ab_small.txt 2>&1
