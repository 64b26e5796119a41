# compute-sanitizer (memcheck / racecheck / synccheck / initcheck) over every kernel variant at small shapes
for tool in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_small.py > gpurun_out/san_$tool.txt 2>&1
  echo "rc=$?" >> gpurun_out/san_$tool.txt
done
tail -3 gpurun_out/san_*.txt
