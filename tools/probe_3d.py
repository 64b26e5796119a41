import os, sys, subprocess, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
# A/B: same schedules with and without the 3-D (one TMA per stage) maps, separate processes
code = r'''
import os, sys
sys.path.insert(0, os.getcwd())
from tools.quick_perf import probe, TC
P = dict(TC, tile_m=256, cluster_m=2, tile_n=256, tile_k=128, stages=3, acc_buffers=2, persistent=1, buffer_c=1, raster_group=16)
probe(8192, 8192, 8192, "bf16", "bf16", [P, dict(P, tile_k=64, stages=6), dict(TC, tile_n=256, stages=4, acc_buffers=2, persistent=1, raster_group=16)], validate=1, repeats=10, rounds=3, cool_s=0.5, cublas=False)
probe(1024, 1024, 1024, "bf16", "bf16", [dict(TC, tile_n=64, stages=8, acc_buffers=2, persistent=1, pack_warps=2), dict(TC, tile_n=64, tile_k=128, stages=4, acc_buffers=2)], validate=1, cublas=False)
'''
for env in ({}, {"XTC_NO_3D_TMA": "1"}):
    print("### env", env, flush=True)
    subprocess.run([sys.executable, "-c", code], env=dict(os.environ, **env))
