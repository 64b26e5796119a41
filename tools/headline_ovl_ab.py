"""Headline A/B: overlapped epilogue (3 stages + 64 KB SMEM tile) vs the 4-stage default."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from quick_perf import probe
from bench import HEADLINE_SCHEDULE as H
V = [dict(H), dict(H, stages=3), dict(H, stages=3, raster_group=16), dict(H, stages=3, raster_group=4)]
probe(8192, 8192, 8192, "bf16", "bf16", V, validate=1, repeats=10, rounds=4, cool_s=0.5)
