"""L14 (32x14x14x256 -> 256, 3x3) A/B: im2col CTA-pair tiles like cuDNN's chosen
cutlass3x_sm100 s256x128 implicit GEMM (pair 256x128, 64-deep stages) vs the pack_halo default.
Interleaved rounds, L2 flushed, median of 30 reps (us)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2512_16512_b200 as xtc
from paper_2512_16512_b200.bench_extras import HALO, PAIR, CONV_SCHEDS
LAYER = sys.argv[1] if len(sys.argv) > 1 else "L14"
if LAYER == "L56":
    from paper_2512_16512_b200.bench_extras import TC
    V = {"halo default": CONV_SCHEDS["L56"][0], "im2col rg8 pw3": CONV_SCHEDS["L56"][2],
         "im2col bres pw3": CONV_SCHEDS["L56"][3]}
    for tk, stg in ((64, 8), (128, 4), (128, 6)):
        for pw in (2, 3):
            V[f"1cta n64 k{tk} s{stg} pw{pw}"] = dict(TC, tile_n=64, tile_k=tk, stages=stg, buffer_c=1, acc_buffers=2,
                                                      persistent=1, pack_warps=pw, raster_group=8)
else:
  V = {"halo default": CONV_SCHEDS["L14"][0], "halo 1cta n128": CONV_SCHEDS["L14"][2]}
for tn in (() if LAYER == "L56" else (128, 256)):
    for tk, stg in ((64, 6), (128, 3), (128, 4)):
        for pers in (0, 1):
            for pw in (2, 3):
                V[f"pair n{tn} k{tk} s{stg} p{pers} pw{pw}"] = dict(PAIR, tile_n=tn, tile_k=tk, stages=stg, buffer_c=1,
                                                                    acc_buffers=1 if (tn == 256 or not pers) else 2,
                                                                    persistent=pers, pack_warps=pw)
st = torch.cuda.current_stream().cuda_stream
H, C = (56, 64) if LAYER == "L56" else (14, 256)
d = xtc.conv2d_desc(32, H, H, C, C, 3, 3, 1, 1, "bf16", "bf16")
x = torch.empty((32, H, H, C), dtype=torch.bfloat16, device="cuda")
w = torch.empty((3, 3, C, C), dtype=torch.bfloat16, device="cuda")
y = torch.empty((32 * H * H, C), dtype=torch.bfloat16, device="cuda")
xtc.xtc_fill(x.data_ptr(), x.numel(), xtc.XTC_BF16, 5, 0, 0, st)
xtc.xtc_fill(w.data_ptr(), w.numel(), xtc.XTC_BF16, 6, 0, 0, st)
ops = []
for name, s in V.items():
    try:
        ops.append((name, xtc.Op(d).apply(xtc.schedule(**s))))
    except xtc.XtcError as e:
        print(f"{name}: illegal ({str(e)[:90]})")
res = {}
for rnd in range(3):
    for name, op in ops:
        m = op.measure(x, w, y, xtc.measure_cfg(warmup=3, repeats=30, flush_l2=1, validate=1 if rnd == 0 else 0,
                                                reuse_reference=1))
        res.setdefault(name, []).append((round(m.t_med_ns / 1e3, 2), round(m.t_mean_ns / 1e3, 2)))
        if rnd == 0 and m.valid != 1:
            res[name].append("INVALID")
for k, v in sorted(res.items(), key=lambda kv: kv[1][-1][1] if isinstance(kv[1][-1], tuple) else 1e9):
    print(f"{k:32s} {v}")
