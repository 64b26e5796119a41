mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q -k "subtiles" > gpurun_out/pytest_msub.log 2>&1; echo rc=$? >> gpurun_out/pytest_msub.log
timeout 600 python tools/headline_msub_ab.py > gpurun_out/headline_msub_ab.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu.log
echo done
