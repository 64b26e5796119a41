set -x
python tools/probe_multicast.py > gpurun_out/probe_mc.json 2>&1
nvidia-smi -q | grep -i -A3 "fabric" > gpurun_out/fabric.txt 2>&1
for tool in memcheck racecheck synccheck initcheck; do
  timeout 600 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_small.py > gpurun_out/san_$tool.txt 2>&1
  echo "rc=$?" >> gpurun_out/san_$tool.txt
done
