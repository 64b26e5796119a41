timeout 900 python -m pytest tests/test_gpu_splitk_cluster.py -x -q -p no:cacheprovider > gpurun_out/t_splitk.log 2>&1; echo rc=$? >> gpurun_out/t_splitk.log
rm -f gpurun_out/trace_*.jsonl
for i in 1 3 6 7; do XTC_TRACE=gpurun_out/trace_$i.jsonl python tools/kernel_time_probe.py $i > /dev/null 2>&1; done
python tools/kernel_time_probe.py > gpurun_out/ktp_events.json 2> gpurun_out/ktp.err
timeout 900 python tools/perf_split_cluster.py > gpurun_out/perf_split.jsonl 2> gpurun_out/perf_split.err
