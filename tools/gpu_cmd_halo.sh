mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 300 -k "halo" > gpurun_out/pytest_halo.log 2>&1; echo rc=$? >> gpurun_out/pytest_halo.log
timeout 300 python tools/halo_probe.py > gpurun_out/halo_probe.log 2>&1
echo done
