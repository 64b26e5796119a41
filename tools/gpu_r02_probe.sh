python tools/probe_symm_multicast.py > gpurun_out/probe_symm.json 2>&1
python tools/kernel_time_probe.py > gpurun_out/ktp_events.json 2> gpurun_out/ktp.err
timeout 900 ncu --metrics gpu__time_duration.sum,sm__cycles_active.max --clock-control none --csv --log-file gpurun_out/ktp_ncu.csv python tools/kernel_time_probe.py > /dev/null 2>&1
for i in 1 2 6 7 5; do XTC_TRACE=gpurun_out/trace_$i.jsonl python tools/kernel_time_probe.py $i > /dev/null 2>&1; done
