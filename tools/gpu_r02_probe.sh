./tools/tma_bench/handoff_bench > gpurun_out/handoff.txt 2>&1
