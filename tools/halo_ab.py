"""A/B the conv_halo variants on one box, in one process (interleaved rounds)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2512_16512_b200 as xtc
base = dict(engine=1, tile_m=128, tile_n=64, tile_k=64, stages=2, swizzle=128, buffer_c=1, acc_buffers=2,
            persistent=1, b_resident=1, pack_halo=1)
variants = [("m128 nbuf2", dict(base), {}), ("m128 nbuf2 wait-all-B", dict(base), {"XTC_DEBUG_SKIP": "256"}),
            ("m128 nbuf3", dict(base), {"XTC_HALO_NBUF": "3"}), ("m128 nbuf1", dict(base), {"XTC_HALO_NBUF": "1"}),
            ("m256 nbuf2", dict(base, tile_m=256), {}), ("m256 nbuf1", dict(base, tile_m=256), {"XTC_HALO_NBUF": "1"}),
            ("m128 nbuf2 no-store-staging", dict(base, buffer_c=0), {}), ("m128 acc1", dict(base, acc_buffers=1), {})]
d = xtc.conv2d_desc(32, 56, 56, 64, 64, 3, 3, 1, 1, "bf16", "bf16")
x = torch.empty((32, 56, 56, 64), dtype=torch.bfloat16, device="cuda"); w = torch.empty((3, 3, 64, 64), dtype=torch.bfloat16, device="cuda")
y = torch.empty((100352, 64), dtype=torch.bfloat16, device="cuda")
st = torch.cuda.current_stream().cuda_stream
xtc.xtc_fill(x.data_ptr(), x.numel(), xtc.XTC_BF16, 5, 0, 0, st); xtc.xtc_fill(w.data_ptr(), w.numel(), xtc.XTC_BF16, 6, 0, 0, st)
ops = []
for name, s, env in variants:
    for k in ("XTC_HALO_NBUF",):
        os.environ.pop(k, None)
    os.environ.update({k: v for k, v in env.items() if k == "XTC_HALO_NBUF"})
    ops.append((name, xtc.Op(d).apply(xtc.schedule(**s)), env))
os.environ.pop("XTC_HALO_NBUF", None)
res = {n: [] for n, _, _ in ops}
for rnd in range(3):
    for name, op, env in ops:
        os.environ["XTC_DEBUG_SKIP"] = env.get("XTC_DEBUG_SKIP", "0")
        m = op.measure(x, w, y, xtc.measure_cfg(warmup=3, repeats=20, flush_l2=1, validate=1 if rnd == 0 else 0, reuse_reference=1))
        res[name].append(round(m.t_med_ns / 1e3, 2))
        if rnd == 0 and m.valid != 1:
            res[name].append("INVALID")
os.environ["XTC_DEBUG_SKIP"] = "0"
for n, v in res.items():
    print(f"{n:32s} {v}")
