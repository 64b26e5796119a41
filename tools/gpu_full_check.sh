# full GPU suite + default bench (the driver's round-end pair)
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/t_all.log 2>&1; tail -3 gpurun_out/t_all.log
timeout 900 python bench.py > gpurun_out/bench.log 2> gpurun_out/bench.err; echo "bench rc=$?"
