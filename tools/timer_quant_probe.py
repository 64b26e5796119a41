"""Event-timer quantisation probe (round 2): per-launch CUDA-event times of the conv layers (L2 flushed
before every launch) for our schedules and cuDNN, 300 reps each -- the distinct values, the median and
the mean.  On the gpurun B200s every single-launch event time is a multiple of ~2.05 us plus jitter, so
medians snap to the grid; the mean over many reps (random start phase) resolves below it.
PYTHONPATH=. python tools/timer_quant_probe.py"""
import collections, json, statistics, sys
import torch
import torch.nn.functional as F
import paper_2512_16512_b200 as xtc
from paper_2512_16512_b200.bench_extras import HALO

REPS = 300
flush = torch.empty(512 * 1024 * 1024 // 4, device="cuda", dtype=torch.float32)


def times(fn):
    for _ in range(5):
        fn()
    ts = []
    for _ in range(REPS):
        flush.sum()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    hist = collections.Counter(round(t, 1) for t in ts)
    return {"med": round(statistics.median(ts), 3), "mean": round(statistics.fmean(ts), 3),
            "top": [v for v, _ in hist.most_common(4)]}


torch.backends.cudnn.benchmark = True
SCHEDS = {"L56": {"pow2-tma": dict(HALO, tile_n=64, stages=2, b_resident=1),
                  "pow2-direct": dict(HALO, tile_n=64, stages=2, b_resident=1, buffer_c=0),
                  "compact": dict(HALO, tile_n=64, stages=2, b_resident=1, pack_halo=2, buffer_c=0)},
          "L14": {"pow2-tma": dict(HALO, tile_n=128, tile_k=128, stages=3)}}
for name, (h, c) in {"L56": (56, 64), "L14": (14, 256)}.items():
    for n in [int(a) for a in sys.argv[1:]] or (32, 8, 1):
        x = torch.randn(n, c, h, h, device="cuda", dtype=torch.bfloat16).to(memory_format=torch.channels_last)
        w = torch.randn(c, c, 3, 3, device="cuda", dtype=torch.bfloat16).to(memory_format=torch.channels_last)
        out = {"layer": name, "n": n, "cudnn": times(lambda: F.conv2d(x, w, padding=1))}
        xn = x.permute(0, 2, 3, 1).contiguous()                      # NHWC
        wn = w.permute(2, 3, 1, 0).contiguous()                      # RSCF
        d = xtc.conv2d_desc(n, h, h, c, c, 3, 3, 1, 1, "bf16", "bf16")
        M, N, K = xtc.gemm_view(d)
        y = torch.empty((M, N), dtype=torch.bfloat16, device="cuda")
        for k, sch in SCHEDS[name].items():
            op = xtc.Op(d).apply(xtc.schedule(**sch))
            out[k] = times(lambda: op.run(xn, wn, y))
        print(json.dumps(out), flush=True)
