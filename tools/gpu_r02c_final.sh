# round-2 end: full GPU suite, smoke, bench line, launch list of the bench, ncu --set full of the headline and the
# conv layers' bench schedules (L56 compact rows, L14 CTA pair), ncu kernel times vs cuDNN
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gputest.log 2>&1; echo rc=$? >> gpurun_out/gputest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo rc=$? >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.log 2> gpurun_out/bench.err; echo rc=$? >> gpurun_out/bench.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02c_launches.csv python bench.py --steps 5 --warmup 3 --no-extras --no-cpu-baseline > /dev/null 2>&1
H='{"engine":1,"tile_m":512,"tile_n":256,"tile_k":64,"stages":3,"swizzle":128,"buffer_c":1,"acc_buffers":1,"persistent":1,"raster_group":8,"order":0,"cluster_m":2}'
timeout 400 ncu --set full --clock-control none --import-source on -k regex:tc_gemm -s 1 -c 1 -o gpurun_out/r02c_headline python tools/run_one.py matmul 8192 8192 8192 bf16 bf16 "$H" 2 > gpurun_out/ncu_h.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:tc_conv_halo -s 1 -c 1 -o gpurun_out/r02c_conv56_compact python tools/run_one.py conv 32 56 56 64 64 bf16 bf16 '{"engine":1,"tile_m":128,"tile_k":64,"swizzle":128,"pack_halo":2,"buffer_c":0,"acc_buffers":2,"persistent":1,"tile_n":64,"stages":2,"b_resident":1}' 2 > gpurun_out/ncu_c56.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:tc_conv_halo -s 1 -c 1 -o gpurun_out/r02c_conv14_pair python tools/run_one.py conv 32 14 14 256 256 bf16 bf16 '{"engine":1,"tile_m":256,"cluster_m":2,"inner_m":256,"tile_k":128,"swizzle":128,"pack_halo":1,"buffer_c":1,"acc_buffers":2,"persistent":1,"tile_n":128,"stages":3}' 2 > gpurun_out/ncu_c14.log 2>&1
REPS=7 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ncu_ab.csv python tools/conv_ncu_ab.py 32 16 8 1 > gpurun_out/ncu_ab_order.txt 2>&1
REPS=7 python tools/ncu_ab_parse.py gpurun_out/ncu_ab.csv gpurun_out/ncu_ab_order.txt > gpurun_out/ncu_ab.txt 2>&1
