"""Headline 8192^3 raster / tile-order A/B: time (sustained-protocol short bursts, interleaved) and DRAM bytes
per launch from the CUPTI counter pass, per (order, raster_group).  PYTHONPATH=. python tools/headline_raster_traffic.py"""
import json
import torch
import paper_2512_16512_b200 as xtc
from bench import HEADLINE_SCHEDULE

dev = torch.device("cuda", 0)
n = 8192
desc = xtc.matmul_desc(n, n, n, "bf16", "bf16")
a = torch.empty((n, n), dtype=torch.bfloat16, device=dev); b = torch.empty_like(a); c = torch.empty_like(a)
s_ = torch.cuda.current_stream().cuda_stream
xtc.xtc_fill(a.data_ptr(), a.numel(), xtc.XTC_BF16, 1, 0, 0, s_); xtc.xtc_fill(b.data_ptr(), b.numel(), xtc.XTC_BF16, 2, 0, 0, s_)
names = ["gpu.dram__bytes_read.sum", "gpu.dram__bytes_write.sum"]
variants = [(o, g) for o in (0, 1) for g in (1, 2, 4, 8, 16, 32)]
res = {v: [] for v in variants}
op = xtc.Op(desc)
for rnd in range(3):
    for o, g in variants:
        sch = dict(HEADLINE_SCHEDULE, order=o, raster_group=g)
        op.apply(xtc.schedule(**sch))
        m = op.measure(a, b, c, xtc.measure_cfg(warmup=3, repeats=15, validate=0), stream=s_)
        res[(o, g)].append(m.t_med_ns / 1e3)
        if rnd == 0:
            cm = op.measure(a, b, c, xtc.measure_cfg(warmup=1, repeats=1, validate=0, counters=names), stream=s_)
            cv = cm.counter_values(names)
            res[(o, g)].append(("dram", (cv[names[0]] + cv[names[1]]) / 1e6 if cv else None))
        torch.cuda.synchronize()
        import time; time.sleep(0.3)
for (o, g), v in res.items():
    ts = [x for x in v if not isinstance(x, tuple)]
    dr = [x[1] for x in v if isinstance(x, tuple)]
    print(json.dumps({"order": o, "raster_group": g, "t_us": sorted(ts), "dram_MB": dr}))
