# epilogue change check: full GPU suite + epilogue phase trace + BASELINE-layer timing
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/t_all.log 2>&1; tail -3 gpurun_out/t_all.log
bash tools/gpu_trace_conv2.sh
PYTHONPATH=. timeout 300 python tools/halo_nbuf_ab.py > gpurun_out/nbuf_ab.log 2>&1
