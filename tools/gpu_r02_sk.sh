timeout 900 python -m pytest tests/test_gpu_stream_k.py -x -q -p no:cacheprovider > gpurun_out/t_sk.log 2>&1; echo rc=$? >> gpurun_out/t_sk.log
timeout 900 python tools/perf_split_cluster.py > gpurun_out/perf_split.jsonl 2> gpurun_out/perf_split.err
