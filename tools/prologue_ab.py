"""A/B of the tcgen05 kernels' prologue order on one box, in one process (interleaved rounds):
early = producers start their TMA while warp 2 allocates TMEM (default),
late  = XTC_DEBUG_LATE_ALLOC=1, the allocation before the prologue barrier (the previous order).
Each config uses its bench_extras best schedule; L2 flushed between timed reps."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2512_16512_b200 as xtc
from paper_2512_16512_b200.bench_extras import MATMUL_SCHEDS, CONV_SCHEDS

dev = torch.device("cuda:0")
st = torch.cuda.current_stream().cuda_stream
cases = []
for n in (512, 1024):
    d = xtc.matmul_desc(n, n, n, "bf16", "bf16")
    cases.append((f"mm{n}", d, MATMUL_SCHEDS[n][0], [(n, n), (n, n)], (n, n)))
for name, (nb, h, c) in {"L56": (32, 56, 64), "L14": (32, 14, 256), "L14n1": (1, 14, 256), "L56n1": (1, 56, 64)}.items():
    d = xtc.conv2d_desc(nb, h, h, c, c, 3, 3, 1, 1, "bf16", "bf16")
    cases.append((name, d, CONV_SCHEDS[name[:3]][0], [(nb, h, h, c), (3, 3, c, c)], (nb * h * h, c)))
ops = []
for name, d, s, shapes, cshape in cases:
    a = torch.empty(shapes[0], dtype=torch.bfloat16, device=dev)
    b = torch.empty(shapes[1], dtype=torch.bfloat16, device=dev)
    c = torch.empty(cshape, dtype=torch.bfloat16, device=dev)
    xtc.xtc_fill(a.data_ptr(), a.numel(), xtc.XTC_BF16, 5, 0, 0, st)
    xtc.xtc_fill(b.data_ptr(), b.numel(), xtc.XTC_BF16, 6, 0, 0, st)
    ops.append((name, xtc.Op(d).apply(xtc.schedule(**s)), (a, b, c)))
res = {}
for rnd in range(4):
    for late in ("0", "1"):
        os.environ["XTC_DEBUG_LATE_ALLOC"] = late
        for name, op, (a, b, c) in ops:
            m = op.measure(a, b, c, xtc.measure_cfg(warmup=3, repeats=30, flush_l2=1, validate=1 if rnd == 0 else 0,
                                                    reuse_reference=1))
            key = f"{name} {'late ' if late == '1' else 'early'}"
            res.setdefault(key, []).append(round(m.t_med_ns / 1e3, 2))
            if rnd == 0 and m.valid != 1:
                res[key].append("INVALID")
for k, v in res.items():
    print(f"{k:16s} {v}")
