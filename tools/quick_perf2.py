import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tools.quick_perf import probe, TC
P = dict(TC, tile_m=256, cluster_m=2)
big = [dict(P, tile_n=256, stages=6, acc_buffers=2, persistent=1, raster_group=8),
       dict(P, tile_n=256, stages=6, acc_buffers=2, persistent=1, raster_group=16),
       dict(P, tile_n=256, stages=6, acc_buffers=2, persistent=1, raster_group=4),
       dict(P, tile_n=256, stages=6, acc_buffers=2, persistent=1, raster_group=8, order=1),
       dict(P, tile_n=256, stages=5, acc_buffers=2, persistent=1, raster_group=8),
       dict(P, tile_n=256, stages=6, acc_buffers=1, persistent=0),
       dict(P, tile_n=192, stages=7, acc_buffers=2, persistent=1, raster_group=8),
       dict(P, tile_n=128, stages=8, acc_buffers=2, persistent=1, raster_group=8),
       dict(TC, tile_n=256, stages=4, acc_buffers=2, persistent=1, raster_group=8)]
probe(8192, 8192, 8192, "bf16", "bf16", big, validate=1, repeats=20)
probe(1024, 1024, 1024, "bf16", "bf16", [dict(P, tile_n=128, stages=6, acc_buffers=2, persistent=1),
                                          dict(P, tile_n=256, stages=6, acc_buffers=2, persistent=1)], validate=1)
