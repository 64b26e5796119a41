mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q -k "cluster_n" > gpurun_out/pytest_cluster.log 2>&1; echo rc=$? >> gpurun_out/pytest_cluster.log
timeout 300 python tools/small_gemm_vs_cublas.py > gpurun_out/small_vs_cublas2.json 2> gpurun_out/small_vs_cublas2.err
echo done
