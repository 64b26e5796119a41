mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q -k "conv" > gpurun_out/pytest_conv.log 2>&1; echo rc=$? >> gpurun_out/pytest_conv.log
timeout 600 python tools/conv14_pair_ab.py L14 > gpurun_out/conv14_ab2.txt 2>&1
timeout 600 python tools/conv14_pair_ab.py L56 > gpurun_out/conv56_ab2.txt 2>&1
echo done
