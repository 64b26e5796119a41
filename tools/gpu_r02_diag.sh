timeout 600 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "halo or conv or cluster or stream" > gpurun_out/t_cl.log 2>&1
P14='{"engine":1,"swizzle":128,"pack_halo":1,"acc_buffers":2,"persistent":1,"tile_m":256,"cluster_m":2,"inner_m":256,"tile_k":128,"tile_n":128,"stages":3,"buffer_c":1}'
P56='{"engine":1,"tile_m":256,"cluster_m":2,"inner_m":256,"tile_k":64,"swizzle":128,"pack_halo":1,"acc_buffers":2,"persistent":1,"tile_n":64,"stages":2,"b_resident":1,"buffer_c":0}'
PYTHONPATH=. timeout 300 python tools/ab_mean.py conv 32 14 256 cudnn "env=0:$P14" "env=8192:$P14" > gpurun_out/ab_early2.txt 2>&1
PYTHONPATH=. timeout 300 python tools/ab_mean.py conv 32 56 64 cudnn "env=0:$P56" "env=8192:$P56" >> gpurun_out/ab_early2.txt 2>&1
PYTHONPATH=. timeout 300 python tools/ab_mean.py conv 1 14 256 cudnn "env=0:$P14" "env=8192:$P14" >> gpurun_out/ab_early2.txt 2>&1
