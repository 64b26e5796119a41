"""Interleaved A/B by the MEAN of many single-launch event times (L2 flushed before each launch), robust to
the ~1 us event-timer grid (profiles/r02c_event_timer_quantisation.txt).  Usage:
  PYTHONPATH=. python tools/ab_mean.py conv B H C  'json-sched' ['json-sched' ...]   (3x3 s1 p1, C -> C, bf16)
  PYTHONPATH=. python tools/ab_mean.py matmul N 'json-sched' ...
  a schedule string 'cudnn' / 'cublas' times the library call on the same operands (context only);
  'env=MASK:json-sched' runs that schedule with XTC_DEBUG_SKIP=MASK (read by the library at each launch)."""
import json, os, statistics, sys
import torch
import torch.nn.functional as F
import paper_2512_16512_b200 as xtc

REPS = 300
torch.backends.cudnn.benchmark = True
flush = torch.empty(512 * 1024 * 1024 // 4, device="cuda", dtype=torch.float32)


def one(fn):
    flush.add_(1.0)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); fn(); e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3


a = sys.argv[1:]
fns, labels = [], []
if a[0] == "conv":
    B, H, C = int(a[1]), int(a[2]), int(a[3])
    x = torch.randn(B, C, H, H, device="cuda", dtype=torch.bfloat16).to(memory_format=torch.channels_last)
    w = torch.randn(C, C, 3, 3, device="cuda", dtype=torch.bfloat16).to(memory_format=torch.channels_last)
    xn, wn = x.permute(0, 2, 3, 1).contiguous(), w.permute(2, 3, 1, 0).contiguous()
    d = xtc.conv2d_desc(B, H, H, C, C, 3, 3, 1, 1, "bf16", "bf16")
    M, N, K = xtc.gemm_view(d)
    y = torch.empty((M, N), dtype=torch.bfloat16, device="cuda")
    for s in a[4:]:
        if s == "cudnn":
            fns.append(lambda: F.conv2d(x, w, padding=1))
        else:
            mask, js = (s[4:].split(":", 1) if s.startswith("env=") else ("0", s))
            op = xtc.Op(d).apply(xtc.schedule(**json.loads(js)))
            fns.append(lambda op=op, mask=mask: (os.environ.__setitem__("XTC_DEBUG_SKIP", mask), op.run(xn, wn, y)))
        labels.append(s)
else:
    n = int(a[1])
    A = torch.randn(n, n, device="cuda", dtype=torch.bfloat16)
    Bm = torch.randn(n, n, device="cuda", dtype=torch.bfloat16)
    Cm = torch.empty_like(A)
    for s in a[2:]:
        if s == "cublas":
            fns.append(lambda: torch.matmul(A, Bm, out=Cm))
        else:
            mask, js = (s[4:].split(":", 1) if s.startswith("env=") else ("0", s))
            op = xtc.Op(xtc.matmul_desc(n, n, n, "bf16", "bf16")).apply(xtc.schedule(**json.loads(js)))
            fns.append(lambda op=op, mask=mask: (os.environ.__setitem__("XTC_DEBUG_SKIP", mask), op.run(A, Bm, Cm)))
        labels.append(s)
for f in fns:
    for _ in range(5):
        f()
ts = [[] for _ in fns]
for _ in range(REPS // 10):
    for i, f in enumerate(fns):
        ts[i] += [one(f) for _ in range(10)]
for lab, t in zip(labels, ts):
    m, se = statistics.fmean(t), statistics.stdev(t) / len(t) ** 0.5
    print(f"{m:8.3f} +- {se:5.3f} us  {lab}", flush=True)
