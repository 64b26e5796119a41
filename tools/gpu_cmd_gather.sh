mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q -k "gather" > gpurun_out/pytest_gather.log 2>&1; echo rc=$? >> gpurun_out/pytest_gather.log
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node=1 --master-addr=127.0.0.1 --master-port=29611 tools/symm_gather_probe.py > gpurun_out/symm_probe.log 2>&1; echo rc=$? >> gpurun_out/symm_probe.log
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-extras --no-cpu-baseline --steps 50 > gpurun_out/bench_quick.log 2> gpurun_out/bench_quick.err
echo done
