mkdir -p gpurun_out; rm -f gpurun_out/trace_cn*.jsonl
A='{"engine":1,"tile_m":128,"tile_n":64,"tile_k":64,"stages":8,"buffer_c":1,"swizzle":128}'
B='{"engine":1,"tile_m":128,"tile_n":64,"tile_k":64,"stages":8,"buffer_c":1,"swizzle":128,"cluster_n":2}'
C='{"engine":1,"tile_m":128,"tile_n":64,"tile_k":64,"stages":8,"buffer_c":1,"swizzle":128,"cluster_n":4}'
XTC_TRACE=gpurun_out/trace_cn1.jsonl python tools/run_one.py matmul 1024 1024 1024 bf16 bf16 "$A" 3 > /dev/null 2>&1
XTC_TRACE=gpurun_out/trace_cn2.jsonl python tools/run_one.py matmul 1024 1024 1024 bf16 bf16 "$B" 3 > /dev/null 2>&1
XTC_TRACE=gpurun_out/trace_cn4.jsonl python tools/run_one.py matmul 1024 1024 1024 bf16 bf16 "$C" 3 > /dev/null 2>&1
for i in 1 2 4; do python tools/trace_report.py gpurun_out/trace_cn$i.jsonl > gpurun_out/trace_cn$i.txt 2>&1; done
timeout 300 ncu --metrics gpu__time_duration.sum,sm__cycles_active.avg,l1tex__m_xbar2l1tex_read_bytes.sum,lts__t_sectors_srcunit_tex.sum --clock-control none --csv --log-file gpurun_out/launches_cn.csv bash -c "python tools/run_one.py matmul 1024 1024 1024 bf16 bf16 '$A' 3; python tools/run_one.py matmul 1024 1024 1024 bf16 bf16 '$B' 3; python tools/run_one.py matmul 1024 1024 1024 bf16 bf16 '$C' 3" > /dev/null 2>&1
echo done
