"""fp32 SIMT schedules at 1024^3 / 512^3 (bench protocol: validated, L2 flushed, means): PYTHONPATH=. python tools/simt_search.py"""
import json
import torch
import paper_2512_16512_b200 as xtc
from paper_2512_16512_b200.bench_extras import _best

dev = torch.device("cuda", 0)
S = lambda **k: dict(engine=0, swizzle=4, stages=2, vector_n=4, **k)
CANDS = [S(tile_m=64, tile_n=64, tile_k=16, inner_m=4, inner_n=4, unroll_k=4),
         S(tile_m=128, tile_n=128, tile_k=8, inner_m=8, inner_n=8, unroll_k=8),
         S(tile_m=128, tile_n=128, tile_k=16, inner_m=8, inner_n=8, unroll_k=8),
         S(tile_m=128, tile_n=64, tile_k=16, inner_m=8, inner_n=8, unroll_k=8),
         S(tile_m=64, tile_n=128, tile_k=16, inner_m=8, inner_n=8, unroll_k=8),
         S(tile_m=64, tile_n=64, tile_k=16, inner_m=8, inner_n=8, unroll_k=8),
         S(tile_m=128, tile_n=64, tile_k=16, inner_m=8, inner_n=4, unroll_k=4),
         S(tile_m=64, tile_n=64, tile_k=32, inner_m=4, inner_n=4, unroll_k=8),
         S(tile_m=128, tile_n=128, tile_k=16, inner_m=8, inner_n=8, unroll_k=8, split_k=2, split_k_mode=0)]
for n in (1024, 512):
    d = xtc.matmul_desc(n, n, n, "f32", "f32")
    r = _best(xtc, torch, dev, d, CANDS, [(n, n), (n, n)], 1669.1)
    print(n, json.dumps({"best_mean_us": r.get("t_mean_us"), "best": r.get("schedule"),
                         "tried": [(t.get("t_mean_us"), t.get("valid"), t.get("illegal")) for t in r["tried"]]}), flush=True)
