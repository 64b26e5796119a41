# Re-entry check after the container was re-created: GPU parity, smoke, bench, reference arm, launch list, halo pair A/B
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo rc=$? >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.log 2> gpurun_out/bench.err; echo rc=$? >> gpurun_out/bench.err
timeout 300 python bench.py --impl reference --steps 2 --warmup 0 > gpurun_out/bench_ref.log 2> gpurun_out/bench_ref.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_headline.csv python bench.py --steps 5 --warmup 3 --no-extras --no-cpu-baseline > /dev/null 2>&1
timeout 600 python tools/halo_pair_ab.py > gpurun_out/halo_pair_ab.txt 2>&1
echo done
