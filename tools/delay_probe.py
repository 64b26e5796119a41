"""measure_impl's per-rep delay budget vs the measured time of short kernels: PYTHONPATH=. python tools/delay_probe.py"""
import os
import torch
import paper_2512_16512_b200 as xtc
from paper_2512_16512_b200.bench_extras import MATMUL_SCHEDS
for n in (1024, 512):
    d = xtc.matmul_desc(n, n, n, "bf16", "bf16")
    a = torch.empty((n, n), dtype=torch.bfloat16, device="cuda"); b = torch.empty_like(a); c = torch.empty_like(a)
    st = torch.cuda.current_stream().cuda_stream
    xtc.xtc_fill(a.data_ptr(), a.numel(), xtc.XTC_BF16, 1, 0, 0, st); xtc.xtc_fill(b.data_ptr(), b.numel(), xtc.XTC_BF16, 2, 0, 0, st)
    for sch in MATMUL_SCHEDS[n][:2]:
        op = xtc.Op(d).apply(xtc.schedule(**sch))
        for rnd in range(2):
            for delay in ("2000", "8000", "30000", "100000"):
                os.environ["XTC_MEASURE_DELAY_NS"] = delay
                m = op.measure(a, b, c, xtc.measure_cfg(warmup=3, repeats=40, flush_l2=1, validate=0))
                print(n, rnd, delay, round(m.t_med_ns / 1e3, 2), round(m.t_mean_ns / 1e3, 2), flush=True)
