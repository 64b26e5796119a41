"""Headline 8192^3 bf16 A/B: the default CTA-pair 256x256 tile vs two M-subtiles per CTA (pair tile
512 x tile_n, as cuBLAS's nvjet 256x256 2cta kernel), interleaved rounds with idles (quick_perf.probe)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from quick_perf import probe
from bench import HEADLINE_SCHEDULE as H
M2 = dict(H, tile_m=512, tile_k=64, stages=4, acc_buffers=1)
V = [dict(H), dict(M2, persistent=0), dict(M2, persistent=1, raster_group=16), dict(M2, persistent=1, raster_group=8),
     dict(M2, persistent=0, raster_group=8), dict(M2, tile_n=128, stages=5, acc_buffers=2, persistent=1, raster_group=16),
     dict(M2, persistent=1, raster_group=16, pack_warps=2)]
probe(8192, 8192, 8192, "bf16", "bf16", V, validate=1, repeats=10, rounds=4, cool_s=0.5)
