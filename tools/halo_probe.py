"""Probe: pack_halo conv schedules vs the im2col kernel on the BASELINE conv configs
(bf16, L2 flushed per rep, validated on chip before timing)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2512_16512_b200 as xtc
from paper_2512_16512_b200.bench_extras import CONV_SCHEDS, TC

H = dict(TC, pack_halo=1, buffer_c=1, persistent=1)
CANDS = {
    "L56": [dict(H, tile_n=64, stages=2, acc_buffers=2, b_resident=1),
            dict(H, tile_m=256, tile_n=64, stages=2, acc_buffers=2, b_resident=1),
            dict(H, tile_n=64, stages=4, acc_buffers=2),
            dict(H, tile_m=256, tile_n=64, stages=4, acc_buffers=2),
            dict(H, tile_n=64, stages=2, acc_buffers=2, b_resident=1, persistent=0)],
    "L14": [dict(H, tile_n=128, stages=4, acc_buffers=2),
            dict(H, tile_n=64, stages=4, acc_buffers=2),
            dict(H, tile_n=128, tile_k=128, stages=3, acc_buffers=2),
            dict(H, tile_n=256, tile_k=64, stages=4, acc_buffers=1),
            dict(H, tile_n=64, tile_k=128, stages=4, acc_buffers=2)],
}
dev = torch.device("cuda:0")
out = {}
for name, (h, c) in {"L56": (56, 64), "L14": (14, 256)}.items():
    for nb in ([int(a) for a in sys.argv[1:]] or [32, 8, 1]):
        d = xtc.conv2d_desc(nb, h, h, c, c, 3, 3, 1, 1, "bf16", "bf16")
        x = torch.empty((nb, h, h, c), dtype=torch.bfloat16, device=dev)
        w = torch.empty((3, 3, c, c), dtype=torch.bfloat16, device=dev)
        M, N, K = xtc.gemm_view(d)
        y = torch.empty((M, N), dtype=torch.bfloat16, device=dev)
        st = torch.cuda.current_stream().cuda_stream
        xtc.xtc_fill(x.data_ptr(), x.numel(), xtc.XTC_BF16, 5, 0, 0, st)
        xtc.xtc_fill(w.data_ptr(), w.numel(), xtc.XTC_BF16, 6, 0, 0, st)
        op = xtc.Op(d)
        rows = []
        for tag, lst in (("halo", CANDS[name]), ("im2col", CONV_SCHEDS[name])):
            for s in lst:
                try:
                    op.apply(xtc.schedule(**s))
                except Exception as e:
                    rows.append({"kind": tag, "err": str(e)[:120], "s": s}); continue
                m = op.measure(x, w, y, xtc.measure_cfg(warmup=3, repeats=20, flush_l2=1, validate=1, reuse_reference=1))
                rows.append({"kind": tag, "valid": m.valid, "t_med_us": round(m.t_med_ns / 1e3, 2),
                             "tflops": round(m.tflops_med, 1), "err": m.max_norm_err, "s": {k: v for k, v in s.items() if k not in TC or s[k] != TC[k]}})
        out[f"{name}_n{nb}"] = rows
        for r in rows:
            print(name, nb, json.dumps(r), flush=True)
json.dump(out, open("gpurun_out/halo_probe.json", "w"), indent=1)
