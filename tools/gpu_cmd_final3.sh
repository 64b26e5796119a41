# end-of-round check on the committed kernels: GPU parity, smoke, 4096-candidate sweep over the widened space, quick bench
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo rc=$? >> gpurun_out/smoke.log
timeout 900 python -m paper_2512_16512_b200.sweep --candidates 4096 > gpurun_out/sweep4096.log 2>&1; echo rc=$? >> gpurun_out/sweep4096.log
timeout 600 python bench.py --steps 50 > gpurun_out/bench_final3.log 2> gpurun_out/bench_final3.err; echo rc=$? >> gpurun_out/bench_final3.err
echo done
