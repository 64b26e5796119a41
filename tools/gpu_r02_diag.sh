export REPS=7
export VARIANTS='{"L56": {"compact": {"engine":1,"tile_m":128,"tile_k":64,"swizzle":128,"pack_halo":2,"buffer_c":0,"acc_buffers":2,"persistent":1,"tile_n":64,"stages":2,"b_resident":1}}, "L14": {"pow2-tma": {"engine":1,"tile_m":128,"tile_k":128,"swizzle":128,"pack_halo":1,"buffer_c":1,"acc_buffers":2,"persistent":1,"tile_n":128,"stages":3}, "pair": {"engine":1,"tile_m":256,"cluster_m":2,"inner_m":256,"tile_k":128,"swizzle":128,"pack_halo":1,"buffer_c":1,"acc_buffers":2,"persistent":1,"tile_n":128,"stages":3}}}'
for m in 0 16384 0 16384; do
XTC_DEBUG_SKIP=$m timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ncu_m$m.csv python tools/conv_ncu_ab.py 32 1 > gpurun_out/ncu_m_order.txt 2>&1
echo "mask $m" >> gpurun_out/ncu_masks.txt
python tools/ncu_ab_parse.py gpurun_out/ncu_m$m.csv gpurun_out/ncu_m_order.txt >> gpurun_out/ncu_masks.txt 2>&1
done
