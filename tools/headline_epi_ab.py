"""Headline A/B: epilogue through SMEM + TMA store (buffer_c 1) vs direct 16-byte stores from the
accumulator registers (buffer_c 0) on the 512x256 pair tile (one TMEM accumulator, so the epilogue
is not overlapped with the next tile's MMAs)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from quick_perf import probe
from bench import HEADLINE_SCHEDULE as H
V = [dict(H), dict(H, buffer_c=0), dict(H, tile_k=128, stages=2), dict(H, tile_k=128, stages=2, buffer_c=0),
     dict(H, buffer_c=0, raster_group=4)]
probe(8192, 8192, 8192, "bf16", "bf16", V, validate=1, repeats=10, rounds=4, cool_s=0.5)
