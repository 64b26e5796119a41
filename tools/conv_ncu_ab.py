"""Conv layers for an ncu launch-duration A/B (round 2): each variant launched REPS times in order, with a
marker kernel (torch.cuda._sleep-free: a tiny fill) between variants so the CSV can be split.  Run under
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file OUT python tools/conv_ncu_ab.py
ncu flushes the caches between kernel replays (cold L2, like the bench protocol) and times each kernel
on the device to the ns, so the ~1 us event-timer quantisation of single launches does not apply."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import torch.nn.functional as F
import paper_2512_16512_b200 as xtc
from paper_2512_16512_b200.bench_extras import HALO

REPS = int(os.environ.get("REPS", "3"))
torch.backends.cudnn.benchmark = True
VARIANTS = json.loads(os.environ.get("VARIANTS", "null")) or {
    "L56": {"pow2-tma": dict(HALO, tile_n=64, stages=2, b_resident=1),
            "compact": dict(HALO, tile_n=64, stages=2, b_resident=1, pack_halo=2, buffer_c=0)},
    "L14": {"pow2-tma": dict(HALO, tile_n=128, tile_k=128, stages=3)}}
marker = torch.empty(1, device="cuda")
order = []
for name, (h, c) in {"L56": (56, 64), "L14": (14, 256)}.items():
    for n in [int(a) for a in sys.argv[1:]] or (32, 8, 1):
        x = torch.randn(n, c, h, h, device="cuda", dtype=torch.bfloat16).to(memory_format=torch.channels_last)
        w = torch.randn(c, c, 3, 3, device="cuda", dtype=torch.bfloat16).to(memory_format=torch.channels_last)
        for _ in range(3):
            F.conv2d(x, w, padding=1)            # cudnn.benchmark picks its algorithm outside the marked region
        torch.cuda.synchronize()
        xn = x.permute(0, 2, 3, 1).contiguous()
        wn = w.permute(2, 3, 1, 0).contiguous()
        d = xtc.conv2d_desc(n, h, h, c, c, 3, 3, 1, 1, "bf16", "bf16")
        M, N, K = xtc.gemm_view(d)
        y = torch.empty((M, N), dtype=torch.bfloat16, device="cuda")
        runs = [("cudnn", lambda: F.conv2d(x, w, padding=1))]
        for k, sch in VARIANTS.get(name, {}).items():
            op = xtc.Op(d).apply(xtc.schedule(**sch))
            runs.append((k, lambda op=op: op.run(xn, wn, y)))
        for k, fn in runs:
            marker.fill_(1.0)
            for _ in range(REPS):
                fn()
            order.append(f"{name}_n{n}:{k}")
        torch.cuda.synchronize()
print(json.dumps(order))
