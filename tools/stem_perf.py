"""Stem conv on the warp-MMA engine: every STEM_MMA_SCHEDS candidate at N = 1, 8, 32, L2 flushed."""
import json
import torch
import paper_2512_16512_b200 as xtc
from paper_2512_16512_b200.bench_extras import STEM_MMA_SCHEDS, _best

dev = torch.device("cuda", 0)
for nb in (1, 8, 32):
    d = xtc.conv2d_desc(nb, 224, 224, 3, 16, 7, 7, 2, 3, "bf16", "bf16")
    r = _best(xtc, torch, dev, d, STEM_MMA_SCHEDS, [(nb, 224, 224, 3), (7, 7, 3, 16)], 1638.9)
    print(json.dumps({"n": nb, "best_us": r.get("t_med_us"), "best": r.get("schedule"), "warm": r.get("warm_l2"),
                      "tried": [(s.get("tile_m"), s.get("pack_halo", 0), s.get("persistent", 0), t)
                                for s, t in zip(STEM_MMA_SCHEDS, r.get("tried", []))]}), flush=True)
