"""fp32 matmul: 3xTF32 tensor-core split vs the SIMT FFMA engine (validated at 1e-5, L2 flushed)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2512_16512_b200 as xtc
from paper_2512_16512_b200.bench_extras import SIMT_SCHEDS, _best
TC = dict(engine=1, tile_m=128, swizzle=128, buffer_c=1)
S3 = [dict(TC, tile_n=128, tile_k=32, stages=3), dict(TC, tile_n=256, tile_k=32, stages=2, persistent=1, acc_buffers=2),
      dict(TC, tile_n=64, tile_k=32, stages=4, persistent=1, acc_buffers=2), dict(TC, tile_n=128, tile_k=64, stages=2),
      dict(TC, tile_n=128, tile_k=32, stages=3, split_k=2)]
dev = torch.device("cuda:0")
for n in (512, 1024, 2048, 4096):
    d = xtc.matmul_desc(n, n, n, "f32", "f32")
    r3 = _best(xtc, torch, dev, d, S3, [(n, n), (n, n)], 1701.1)
    rs = _best(xtc, torch, dev, d, SIMT_SCHEDS, [(n, n), (n, n)], 1701.1)
    print(n, json.dumps({"3xtf32": {k: r3.get(k) for k in ("tflops_med", "t_med_us", "max_norm_err", "schedule")},
                         "simt": {k: rs.get(k) for k in ("tflops_med", "t_med_us", "max_norm_err")},
                         "tried3": r3.get("tried")}), flush=True)
