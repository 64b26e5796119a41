"""Probe one pack_halo schedule in its own process (a fault kills only this case): python tools/compact_probe.py 'json' B H W C F"""
import json, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import paper_2512_16512_b200 as xtc
from gpu_util import run_conv
from seeded_inputs import MODE_INT
sch = json.loads(sys.argv[1])
B, H, W, C, F = (int(a) for a in sys.argv[2:7])
d = xtc.conv2d_desc(B, H, W, C, F, 3, 3, 1, 1, "bf16", "bf16")
try:
    run_conv(d, "bf16", "bf16", xtc.schedule(**sch), MODE_INT)
    print("OK", sys.argv[1:])
except Exception as e:
    print("FAIL", sys.argv[1:], repr(e)[:300])
