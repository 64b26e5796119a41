"""A/B of the pack_halo conv on one box, interleaved rounds: 1-CTA tiles vs the CTA pair
(inner_m 256, cta_group::2) on the BASELINE L14 layer (and L14 at N=1, 8; a 28x28 layer)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2512_16512_b200 as xtc
from paper_2512_16512_b200.bench_extras import HALO
PAIR = dict(HALO, tile_m=256, cluster_m=2, inner_m=256)
variants = {
    "1cta n128 k128 s3": dict(HALO, tile_n=128, tile_k=128, stages=3),
    "1cta n64 k128 s4": dict(HALO, tile_n=64, tile_k=128, stages=4),
    "1cta n128 k256 s2": dict(HALO, tile_n=128, tile_k=256, stages=2),
    "pair n128 k128 s3": dict(PAIR, tile_n=128, tile_k=128, stages=3),
    "pair n128 k128 s5": dict(PAIR, tile_n=128, tile_k=128, stages=5),
    "pair n128 k128 s6 dc": dict(PAIR, tile_n=128, tile_k=128, stages=6, buffer_c=0),
    "pair n128 k256 s3": dict(PAIR, tile_n=128, tile_k=256, stages=3),
    "pair n128 k256 s4 dc": dict(PAIR, tile_n=128, tile_k=256, stages=4, buffer_c=0),
    "pair n256 k256 s2": dict(PAIR, tile_n=256, tile_k=256, stages=2),
}
shapes = {"L14 n32": (32, 14, 256, 256), "L14 n8": (8, 14, 256, 256), "L14 n1": (1, 14, 256, 256),
          "28x28x128 n32": (32, 28, 128, 128)}
st = torch.cuda.current_stream().cuda_stream
ops = []
for sname, (nb, h, c, f) in shapes.items():
    d = xtc.conv2d_desc(nb, h, h, c, f, 3, 3, 1, 1, "bf16", "bf16")
    x = torch.empty((nb, h, h, c), dtype=torch.bfloat16, device="cuda")
    w = torch.empty((3, 3, c, f), dtype=torch.bfloat16, device="cuda")
    y = torch.empty((nb * h * h, f), dtype=torch.bfloat16, device="cuda")
    xtc.xtc_fill(x.data_ptr(), x.numel(), xtc.XTC_BF16, 5, 0, 0, st)
    xtc.xtc_fill(w.data_ptr(), w.numel(), xtc.XTC_BF16, 6, 0, 0, st)
    for vname, s in variants.items():
        try:
            ops.append((f"{sname:14s} {vname}", xtc.Op(d).apply(xtc.schedule(**s)), (x, w, y)))
        except xtc.XtcError as e:
            print(f"{sname:14s} {vname}: illegal ({str(e)[:80]})")
res = {}
for rnd in range(3):
    for name, op, (x, w, y) in ops:
        m = op.measure(x, w, y, xtc.measure_cfg(warmup=3, repeats=30, flush_l2=1, validate=1 if rnd == 0 else 0,
                                                reuse_reference=1))
        res.setdefault(name, []).append(round(m.t_med_ns / 1e3, 2))
        if rnd == 0 and m.valid != 1:
            res[name].append("INVALID")
for k, v in res.items():
    print(f"{k:34s} {v}")
