"""Interleaved A/B of conv schedules on the BASELINE layers (L2 flushed): PYTHONPATH=. python tools/conv_ab.py"""
import json, sys
import torch
import paper_2512_16512_b200 as xtc
from paper_2512_16512_b200.bench_extras import HALO, TC, _best

dev = torch.device("cuda", 0)
CANDS = {
    "L56": [dict(HALO, tile_n=64, stages=2, b_resident=1),
            dict(HALO, tile_n=64, stages=2, b_resident=1, buffer_c=0),
            dict(HALO, tile_n=64, stages=2, b_resident=1, pack_halo=2, buffer_c=0),
            dict(HALO, tile_m=256, tile_n=64, stages=2, b_resident=1, pack_halo=2, buffer_c=0)],
    "L14": [dict(HALO, tile_n=128, tile_k=128, stages=3)],
}
LAYERS = {"L56": (56, 64), "L14": (14, 256)}
for rnd in range(2):
    for name, (hw, c) in LAYERS.items():
        for nb in ([int(a) for a in sys.argv[1:]] or [1, 8, 32]):
            d = xtc.conv2d_desc(nb, hw, hw, c, c, 3, 3, 1, 1, "bf16", "bf16")
            r = _best(xtc, torch, dev, d, CANDS[name], [(nb, hw, hw, c), (3, 3, c, c)], 1638.9)
            print(json.dumps({"round": rnd, "layer": name, "n": nb, "best_us": r.get("t_med_us"),
                              "tried": [t.get("t_med_us", t.get("illegal")) for t in r.get("tried", [])]}), flush=True)
