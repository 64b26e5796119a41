# round 2: cluster split-K parity + sanitizer + multicast probe + perf A/B
python tools/probe_multicast.py > gpurun_out/probe_mc.json 2>&1
timeout 900 python -m pytest tests/test_gpu_splitk_cluster.py -x -q -p no:cacheprovider > gpurun_out/t_splitk.log 2>&1; echo rc=$? >> gpurun_out/t_splitk.log
for tool in synccheck racecheck; do
  timeout 600 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_small.py > gpurun_out/san_$tool.txt 2>&1
  echo "rc=$?" >> gpurun_out/san_$tool.txt
done
timeout 900 python tools/perf_split_cluster.py > gpurun_out/perf_split.jsonl 2> gpurun_out/perf_split.err
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gputest.log 2>&1; echo rc=$? >> gpurun_out/gputest.log
