mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 300 -k "counter" > gpurun_out/pytest_counters.log 2>&1; echo rc=$? >> gpurun_out/pytest_counters.log
timeout 300 python - > gpurun_out/counters_demo.log 2>&1 <<'PY'
import torch, json
import paper_2512_16512_b200 as xtc
n = 8192
desc = xtc.matmul_desc(n, n, n, "bf16", "bf16")
a = torch.empty((n, n), dtype=torch.bfloat16, device="cuda:0"); b = torch.empty_like(a); c = torch.empty_like(a)
st = torch.cuda.current_stream().cuda_stream
xtc.xtc_fill(a.data_ptr(), a.numel(), xtc.XTC_BF16, 1, 0, 0, st); xtc.xtc_fill(b.data_ptr(), b.numel(), xtc.XTC_BF16, 2, 0, 0, st)
op = xtc.Op(desc)
import bench
op.apply(xtc.schedule(**bench.HEADLINE_SCHEDULE))
names = ["gpu.dram__bytes_read.sum", "gpu.dram__bytes_write.sum", "gpu.gpu__time_duration.sum",
         "gpu.sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
         "gpu.sm__throughput.avg.pct_of_peak_sustained_elapsed", "gpu.dram__throughput.avg.pct_of_peak_sustained_elapsed"]
m = op.measure(a, b, c, xtc.measure_cfg(warmup=3, repeats=10, flush_l2=1, validate=1, counters=names, peak_tflops=1701.1))
print(json.dumps({"valid": m.valid, "tflops_med": m.tflops_med, "n_counters": m.n_counters, "err": xtc.xtc_last_error() if m.n_counters < 0 else "",
                  "counters": m.counter_values(names)}, indent=1))
PY
echo done
