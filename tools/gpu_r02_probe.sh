rm -f gpurun_out/trace_*.jsonl
python tools/kernel_time_probe.py 4 10 11 12 > gpurun_out/ktp_events.json 2> gpurun_out/ktp.err
XTC_SK_NOCOOP=1 python tools/kernel_time_probe.py 4 10 11 12 > gpurun_out/ktp_events_nocoop.json 2>> gpurun_out/ktp.err
for i in 10 11; do XTC_TRACE=gpurun_out/trace_$i.jsonl python tools/kernel_time_probe.py $i > /dev/null 2>&1; done
timeout 600 ncu --metrics gpu__time_duration.sum,sm__cycles_active.max --clock-control none --csv --log-file gpurun_out/ktp_ncu.csv python tools/kernel_time_probe.py 10 11 > /dev/null 2>&1
