# round-1 final (2): GPU parity, smoke, bench line, reference arm, launch list, headline ncu capture
mkdir -p gpurun_out
P='{"engine":1,"tile_m":512,"tile_n":256,"tile_k":64,"stages":3,"swizzle":128,"buffer_c":1,"acc_buffers":1,"persistent":1,"raster_group":8,"order":0,"cluster_m":2}'
# (GPU parity ran just before on the same code)
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo rc=$? >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.log 2> gpurun_out/bench.err; echo rc=$? >> gpurun_out/bench.err
timeout 300 python bench.py --impl reference --steps 2 --warmup 0 > gpurun_out/bench_ref.log 2> gpurun_out/bench_ref.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_final7.csv python bench.py --steps 5 --warmup 3 --no-extras --no-cpu-baseline > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:tc_gemm -s 1 -c 1 -o gpurun_out/prof_headline_final7 -f python tools/run_one.py matmul 8192 8192 8192 bf16 bf16 "$P" 2 > gpurun_out/ncu_final7.log 2>&1
echo done
