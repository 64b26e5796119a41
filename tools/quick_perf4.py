import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tools.quick_perf import probe, TC
P = dict(TC, tile_m=256, cluster_m=2, tile_n=256, acc_buffers=2, persistent=1)
big = [dict(P, stages=6, buffer_c=1, raster_group=16),
       dict(P, stages=3, tile_k=128, buffer_c=1, raster_group=16),
       dict(P, stages=7, buffer_c=0, raster_group=16),
       dict(P, stages=3, tile_k=128, buffer_c=0, raster_group=16),
       dict(P, stages=6, buffer_c=1, raster_group=8),
       dict(TC, tile_n=256, stages=4, acc_buffers=2, persistent=1, raster_group=16, buffer_c=1)]
probe(8192, 8192, 8192, "bf16", "bf16", big, validate=1, repeats=30)
probe(4096, 4096, 4096, "bf16", "bf16", big[:2], validate=1, repeats=30)
probe(1024, 1024, 1024, "bf16", "bf16", [dict(TC, tile_n=64, stages=8, acc_buffers=2, persistent=1, buffer_c=1),
                                          dict(TC, tile_n=128, stages=6, acc_buffers=2, persistent=1, buffer_c=1)], validate=1)
