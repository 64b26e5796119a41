mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 300 -k "halo" > gpurun_out/pytest_halo.log 2>&1; echo rc=$? >> gpurun_out/pytest_halo.log
H='{"engine":1,"tile_m":256,"tile_n":64,"tile_k":64,"stages":2,"swizzle":128,"buffer_c":1,"acc_buffers":2,"persistent":1,"b_resident":1,"pack_halo":1}'
timeout 300 python tools/halo_diag.py "$H" > gpurun_out/halo_diag.log 2>&1
timeout 300 python tools/halo_probe.py 32 > gpurun_out/halo_probe.log 2>&1
echo done
