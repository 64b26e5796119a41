# 2-rank rehearsal of bench.py N>1 on one GPU (gloo + symmetric memory), fused and NCCL-form gathers
mkdir -p gpurun_out
for g in fused nccl; do
XTC_BENCH_DIST=gloo-shared timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1 --master-port=2955$([ $g = fused ] && echo 1 || echo 2) bench.py --gpus 2 --steps 5 --warmup 3 --no-cpu-baseline --no-extras --gather $g > gpurun_out/rehearsal_$g.log 2> gpurun_out/rehearsal_$g.err; echo rc=$? >> gpurun_out/rehearsal_$g.err
done
echo done
