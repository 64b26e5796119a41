import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tools.quick_perf import probe, TC
P = dict(TC, tile_m=256, cluster_m=2, tile_n=256, acc_buffers=2, persistent=1)
big = [dict(P, stages=6, buffer_c=1, raster_group=16),
       dict(P, stages=7, buffer_c=0, raster_group=16),
       dict(P, stages=7, buffer_c=0, raster_group=8),
       dict(P, stages=6, buffer_c=0, raster_group=16),
       dict(P, stages=7, buffer_c=0, raster_group=12),
       dict(P, stages=3, tile_k=128, buffer_c=0, raster_group=16)]
probe(8192, 8192, 8192, "bf16", "bf16", big, validate=1, repeats=30)
