"""Headline A/B round 2: raster / order / depth around the two-M-subtile pair tile (512 x 256)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from quick_perf import probe
from bench import HEADLINE_SCHEDULE as H
M2 = dict(H, tile_m=512, tile_k=64, stages=4, acc_buffers=1, persistent=1)
V = [dict(H), dict(M2, raster_group=8), dict(M2, raster_group=4), dict(M2, raster_group=2), dict(M2, raster_group=6),
     dict(M2, raster_group=8, order=1), dict(M2, raster_group=4, order=1), dict(M2, raster_group=8, tile_k=128, stages=2),
     dict(M2, tile_n=128, acc_buffers=2, raster_group=8)]
probe(8192, 8192, 8192, "bf16", "bf16", V, validate=0, repeats=10, rounds=4, cool_s=0.5)
