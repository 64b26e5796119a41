P='"engine":1,"tile_m":256,"cluster_m":2,"inner_m":256,"tile_k":64,"swizzle":128,"acc_buffers":2,"persistent":1,"tile_n":64,"buffer_c":0'
timeout 60 python tools/compact_probe.py "{$P,\"stages\":2,\"b_resident\":1,\"pack_halo\":2}" 4 56 56 64 64 > gpurun_out/probe_pc.txt 2>&1
grep -q "^OK" gpurun_out/probe_pc.txt && timeout 600 python -m pytest tests -m gpu -q -p no:cacheprovider -k "halo or conv" > gpurun_out/t_pc.log 2>&1
L56C='{"engine":1,"tile_m":128,"tile_k":64,"swizzle":128,"pack_halo":2,"buffer_c":0,"acc_buffers":2,"persistent":1,"tile_n":64,"stages":2,"b_resident":1}'
for n in 32 16 8; do
grep -q "^OK" gpurun_out/probe_pc.txt && PYTHONPATH=. timeout 300 python tools/ab_mean.py conv $n 56 64 cudnn "$L56C" "{$P,\"stages\":2,\"b_resident\":1,\"pack_halo\":1}" "{$P,\"stages\":2,\"b_resident\":1,\"pack_halo\":2}" >> gpurun_out/ab_pc.txt 2>&1
done
