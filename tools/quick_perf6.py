import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tools.conv_diag import bench
import paper_2512_16512_b200 as xtc
TC = dict(engine=1, tile_m=128, tile_k=64, swizzle=128, buffer_c=1)
d = xtc.conv2d_desc(32, 56, 56, 64, 64)
for s in [dict(TC, tile_n=64, stages=8, acc_buffers=2, persistent=1, pack_warps=3),
          dict(TC, tile_n=64, stages=7, acc_buffers=2, persistent=1, pack_warps=3, b_resident=1),
          dict(TC, tile_n=64, stages=6, acc_buffers=2, persistent=1, pack_warps=2, b_resident=1),
          dict(TC, tile_n=64, stages=7, acc_buffers=2, persistent=1, pack_warps=1, b_resident=1),
          dict(TC, tile_n=64, stages=7, acc_buffers=2, persistent=1, pack_warps=3, b_resident=1, raster_group=4),
          dict(TC, tile_n=64, tile_k=128, stages=3, acc_buffers=2, persistent=1, pack_warps=3, b_resident=1)]:
    print(json.dumps({"layer": "L56", "sch": {k: v for k, v in s.items() if k not in ("engine", "swizzle", "tile_m")},
                      "conv": bench(d, [(32, 56, 56, 64), (3, 3, 64, 64)], s)}), flush=True)
