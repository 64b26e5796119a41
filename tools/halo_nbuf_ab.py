"""A/B of the conv_halo patch-buffer count (XTC_HALO_NBUF) on the BASELINE conv layers, L2 flushed,
interleaved rounds.  PYTHONPATH=. python tools/halo_nbuf_ab.py"""
import json, os
import torch
import paper_2512_16512_b200 as xtc
from paper_2512_16512_b200.bench_extras import CONV_SCHEDS, _best

dev = torch.device("cuda", 0)
LAYERS = {"L56": (56, 64), "L14": (14, 256)}
for rnd in range(1):
    for name, (hw, c) in LAYERS.items():
        for nb in (1, 8, 32):
            for nbuf in ("2", "3"):
                os.environ["XTC_HALO_NBUF"] = nbuf
                d = xtc.conv2d_desc(nb, hw, hw, c, c, 3, 3, 1, 1, "bf16", "bf16")
                r = _best(xtc, torch, dev, d, [s for s in CONV_SCHEDS[name] if s.get("pack_halo")],
                          [(nb, hw, hw, c), (3, 3, c, c)], 1638.9)
                print(json.dumps({"round": rnd, "layer": name, "n": nb, "nbuf": nbuf, "best_us": r.get("t_med_us"),
                                  "tried": [t.get("t_med_us") for t in r.get("tried", [])]}), flush=True)
