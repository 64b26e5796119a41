mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 600 -x > gpurun_out/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu.log
timeout 300 python -m paper_2512_16512_b200.sweep --candidates 4096 --out gpurun_out/sweep4096.json > gpurun_out/sweep4096.log 2>&1
timeout 300 python -m paper_2512_16512_b200.sweep --candidates 1024 --engine simt --out gpurun_out/sweep_simt1024.json > gpurun_out/sweep_simt.log 2>&1
timeout 300 python -m paper_2512_16512_b200.sweep --candidates 1024 --m 512 --n 512 --k 512 --out gpurun_out/sweep512.json > gpurun_out/sweep512.log 2>&1
echo done
