mkdir -p gpurun_out
./tools/umma_shift/umma_shift > gpurun_out/umma_shift.log 2>&1
timeout 300 python tools/cudnn_conv_ref.py > gpurun_out/cudnn_conv.log 2>&1
echo done
