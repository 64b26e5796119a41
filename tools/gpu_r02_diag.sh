timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ncu_ab.csv python tools/conv_ncu_ab.py 32 16 8 1 > gpurun_out/ncu_ab_order.txt 2>&1
python tools/ncu_ab_parse.py gpurun_out/ncu_ab.csv gpurun_out/ncu_ab_order.txt > gpurun_out/ncu_ab.txt 2>&1
