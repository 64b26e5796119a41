"""Headline 8192^3 bf16 schedule A/B (interleaved rounds, cool-down idles; tools/quick_perf.probe):
raster group / order / stage depth around the bench.py default."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from quick_perf import probe
from bench import HEADLINE_SCHEDULE as H
V = [dict(H), dict(H, raster_group=8), dict(H, raster_group=12), dict(H, raster_group=24), dict(H, raster_group=32),
     dict(H, order=1), dict(H, order=1, raster_group=8), dict(H, tile_k=64, stages=6), dict(H, pack_warps=2)]
probe(8192, 8192, 8192, "bf16", "bf16", V, repeats=10, rounds=4, cool_s=0.5)
