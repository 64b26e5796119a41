"""Headline A/B: 512x256 pair tile with 4 stages + 2 epilogue staging buffers per warp vs 3 stages +
4 buffers (more TMA stores in flight while the single accumulator drains)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from quick_perf import probe
from bench import HEADLINE_SCHEDULE as H
V = [dict(H), dict(H, stages=3), dict(H, stages=3, raster_group=16), dict(H, stages=3, pack_warps=2)]
probe(8192, 8192, 8192, "bf16", "bf16", V, validate=1, repeats=10, rounds=4, cool_s=0.5)
