import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tools.quick_perf import probe
S = dict(engine=0, swizzle=4, stages=2, vector_n=4)
sch = [dict(S, tile_m=128, tile_n=128, tile_k=16, inner_m=8, inner_n=8, unroll_k=4),
       dict(S, tile_m=128, tile_n=128, tile_k=16, inner_m=8, inner_n=8, unroll_k=1),
       dict(S, tile_m=128, tile_n=64, tile_k=16, inner_m=8, inner_n=4, unroll_k=4),
       dict(S, tile_m=64, tile_n=128, tile_k=16, inner_m=4, inner_n=8, unroll_k=4),
       dict(S, tile_m=128, tile_n=64, tile_k=32, inner_m=8, inner_n=4, unroll_k=8),
       dict(S, tile_m=64, tile_n=64, tile_k=16, inner_m=4, inner_n=4, unroll_k=4)]
probe(4096, 4096, 4096, "f32", "f32", sch, validate=1, repeats=5, rounds=2)
probe(1024, 1024, 1024, "f32", "f32", sch, validate=1, repeats=10, rounds=2)
