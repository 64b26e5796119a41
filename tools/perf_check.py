"""Quick perf check of the main configs (validated, L2 flushed; medians), one process."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2512_16512_b200 as xtc
import bench
from paper_2512_16512_b200.bench_extras import MATMUL_SCHEDS, CONV_SCHEDS, SIMT_SCHEDS, _best
dev = torch.device("cuda:0")
peak = 1701.1
out = {}
n = 8192
d = xtc.matmul_desc(n, n, n, "bf16", "bf16")
out["mm8192_headline"] = _best(xtc, torch, dev, d, [bench.HEADLINE_SCHEDULE], [(n, n), (n, n)], peak, flush=0)
for n in (1024, 512):
    d = xtc.matmul_desc(n, n, n, "bf16", "bf16")
    out[f"mm{n}"] = _best(xtc, torch, dev, d, MATMUL_SCHEDS[n], [(n, n), (n, n)], peak)
for name, (h, c) in {"L56": (56, 64), "L14": (14, 256)}.items():
    d = xtc.conv2d_desc(32, h, h, c, c, 3, 3, 1, 1, "bf16", "bf16")
    out[f"conv_{name}"] = _best(xtc, torch, dev, d, CONV_SCHEDS[name], [(32, h, h, c), (3, 3, c, c)], peak)
for k, v in out.items():
    print(k, json.dumps({"best_us": round(v.get("t_med_us", -1), 2), "tflops": round(v.get("tflops_med", -1), 1),
                         "tried": v.get("tried")}))
