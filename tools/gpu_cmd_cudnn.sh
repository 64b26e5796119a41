mkdir -p gpurun_out
timeout 300 ncu --metrics gpu__time_duration.sum,launch__grid_size,launch__cluster_dim_x,launch__shared_mem_per_block_dynamic,launch__block_size --clock-control none --csv --log-file gpurun_out/launches_cudnn14.csv python tools/cudnn_conv_one.py 32 14 256 > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum,launch__grid_size,launch__cluster_dim_x,launch__shared_mem_per_block_dynamic,launch__block_size --clock-control none --csv --log-file gpurun_out/launches_cudnn56.csv python tools/cudnn_conv_one.py 32 56 64 > /dev/null 2>&1
echo done
