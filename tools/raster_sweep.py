import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tools.quick_perf import probe, TC
P = dict(TC, tile_m=256, cluster_m=2, tile_n=256, tile_k=128, stages=3, acc_buffers=2, persistent=1, buffer_c=1)
scheds = [dict(P, raster_group=g, order=o) for o in (0, 1) for g in (4, 6, 8, 12, 16, 32)]
scheds += [dict(P, raster_group=16, pack_warps=2), dict(P, raster_group=6, pack_warps=2)]
probe(8192, 8192, 8192, "bf16", "bf16", scheds, validate=1, repeats=10, rounds=4, cool_s=0.5)
