"""Diagnose the pack_halo conv pipeline: time the kernel with parts switched off
(XTC_DEBUG_SKIP mask: 1 no MMAs, 2 no patch TMA, 4 no output stores) and trace one
launch per variant.  Output is invalid for every mask != 0 (diagnostics only)."""
import json, os, subprocess, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2512_16512_b200 as xtc
sch = json.loads(sys.argv[1])
nb, h, c = (int(a) for a in sys.argv[2:5]) if len(sys.argv) > 4 else (32, 56, 64)
d = xtc.conv2d_desc(nb, h, h, c, c, 3, 3, 1, 1, "bf16", "bf16")
x = torch.empty((nb, h, h, c), dtype=torch.bfloat16, device="cuda")
w = torch.empty((3, 3, c, c), dtype=torch.bfloat16, device="cuda")
M, N, K = xtc.gemm_view(d)
y = torch.empty((M, N), dtype=torch.bfloat16, device="cuda")
st = torch.cuda.current_stream().cuda_stream
xtc.xtc_fill(x.data_ptr(), x.numel(), xtc.XTC_BF16, 5, 0, 0, st)
xtc.xtc_fill(w.data_ptr(), w.numel(), xtc.XTC_BF16, 6, 0, 0, st)
op = xtc.Op(d).apply(xtc.schedule(**sch))
for mask in [int(v) for v in os.environ.get("DIAG_MASKS", "0,1,2,4,6,3,5,7").split(",")]:
    os.environ["XTC_DEBUG_SKIP"] = str(mask)
    for flush in (1, 0):
        m = op.measure(x, w, y, xtc.measure_cfg(warmup=3, repeats=20, flush_l2=flush, validate=0))
        print(f"mask {mask} flush {flush}: t_med {m.t_med_ns / 1e3:.2f} us  ({m.tflops_med:.0f} TF/s)", flush=True)
os.environ["XTC_DEBUG_SKIP"] = "0"
