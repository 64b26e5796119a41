import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tools.quick_perf import probe, TC
from tools.conv_diag import bench
import paper_2512_16512_b200 as xtc
P = dict(TC, tile_m=256, cluster_m=2, tile_n=256, acc_buffers=2, persistent=1, raster_group=16, buffer_c=1)
probe(8192, 8192, 8192, "bf16", "bf16", [dict(P, tile_k=128, stages=3, pack_warps=w) for w in (1, 2, 3)] +
      [dict(P, tile_k=64, stages=6, pack_warps=w) for w in (2, 3)], validate=1, repeats=30)
probe(1024, 1024, 1024, "bf16", "bf16", [dict(TC, tile_n=64, stages=8, acc_buffers=2, persistent=1, buffer_c=1, pack_warps=w) for w in (1, 2, 3)], validate=1)
for name, (B, H, C, F) in {"L56": (32, 56, 64, 64), "L14": (32, 14, 256, 256)}.items():
    d = xtc.conv2d_desc(B, H, H, C, F)
    for w in (1, 2, 3):
        s = dict(TC, tile_n=min(F, 256), stages=8 if F == 64 else 4, acc_buffers=2, persistent=1, raster_group=8, buffer_c=1, pack_warps=w)
        print(json.dumps({"layer": name, "pack_warps": w, "conv": bench(d, [(B, H, H, C), (3, 3, C, F)], s)}), flush=True)
        if F >= 128:
            s2 = dict(TC, tile_m=256, cluster_m=2, tile_n=256, tile_k=128, stages=3, acc_buffers=2, persistent=1, buffer_c=1, pack_warps=w)
            print(json.dumps({"layer": name + "_pair", "pack_warps": w, "conv": bench(d, [(B, H, H, C), (3, 3, C, F)], s2)}), flush=True)
