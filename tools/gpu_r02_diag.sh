H='"engine":1,"swizzle":128,"pack_halo":1,"acc_buffers":2,"persistent":1,"tile_m":128'
PYTHONPATH=. timeout 300 python tools/ab_mean.py conv 1 14 256 cudnn \
 "{$H,\"tile_k\":128,\"tile_n\":64,\"stages\":4,\"buffer_c\":0}" \
 "{$H,\"tile_k\":64,\"tile_n\":64,\"stages\":8,\"buffer_c\":0}" \
 "{$H,\"tile_k\":64,\"tile_n\":64,\"stages\":12,\"buffer_c\":0}" \
 "{$H,\"tile_k\":128,\"tile_n\":64,\"stages\":6,\"buffer_c\":0}" \
 "{$H,\"tile_k\":64,\"tile_n\":128,\"stages\":8,\"buffer_c\":0}" > gpurun_out/ab14_1b.txt 2>&1
PYTHONPATH=. timeout 300 python tools/ab_mean.py conv 8 14 256 cudnn \
 "{$H,\"tile_k\":128,\"tile_n\":64,\"stages\":4,\"buffer_c\":0}" \
 "{$H,\"tile_k\":64,\"tile_n\":64,\"stages\":8,\"buffer_c\":0}" \
 "{$H,\"tile_k\":128,\"tile_n\":64,\"stages\":6,\"buffer_c\":0}" > gpurun_out/ab14_8b.txt 2>&1
