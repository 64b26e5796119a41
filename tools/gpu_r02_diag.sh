M512='{"engine":1,"tile_m":128,"tile_k":128,"swizzle":128,"tile_n":64,"stages":4,"buffer_c":1,"acc_buffers":1,"pack_warps":2}'
M1024='{"engine":1,"tile_m":128,"tile_k":128,"swizzle":128,"tile_n":64,"stages":3,"buffer_c":1,"acc_buffers":2,"persistent":0,"raster_group":2}'
L14='{"engine":1,"swizzle":128,"pack_halo":1,"acc_buffers":2,"persistent":1,"tile_m":256,"cluster_m":2,"inner_m":256,"tile_k":128,"tile_n":128,"stages":3,"buffer_c":1}'
L56='{"engine":1,"tile_m":128,"tile_k":64,"swizzle":128,"pack_halo":1,"buffer_c":1,"acc_buffers":2,"persistent":1,"tile_n":64,"stages":2,"b_resident":1}'
PYTHONPATH=. timeout 200 python tools/ab_mean.py matmul 512 cublas "env=0:$M512" "env=65536:$M512" > gpurun_out/abx.txt 2>&1
PYTHONPATH=. timeout 200 python tools/ab_mean.py matmul 1024 cublas "env=0:$M1024" "env=65536:$M1024" >> gpurun_out/abx.txt 2>&1
PYTHONPATH=. timeout 200 python tools/ab_mean.py conv 32 14 256 cudnn "env=0:$L14" "env=65536:$L14" >> gpurun_out/abx.txt 2>&1
PYTHONPATH=. timeout 200 python tools/ab_mean.py conv 1 56 64 cudnn "env=0:$L56" "env=65536:$L56" >> gpurun_out/abx.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "halo or conv or overlapped or many_tiles or fullsize" > gpurun_out/t_x.log 2>&1
