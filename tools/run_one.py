"""Run one op/schedule a few times (for ncu captures).  Usage:
  python tools/run_one.py matmul M N K in out 'json-schedule' [reps]
  python tools/run_one.py conv B H W C F in out 'json-schedule' [reps]"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2512_16512_b200 as xtc
T = {"bf16": torch.bfloat16, "f32": torch.float32, "tf32": torch.float32}
a = sys.argv[1:]
if a[0] == "matmul":
    M, N, K = map(int, a[1:4]); ind, outd, sch = a[4], a[5], json.loads(a[6]); reps = int(a[7]) if len(a) > 7 else 3
    d = xtc.matmul_desc(M, N, K, ind, outd); sa, sb = (M, K), (K, N)
else:
    B, H, W, C, F = map(int, a[1:6]); ind, outd, sch = a[6], a[7], json.loads(a[8]); reps = int(a[9]) if len(a) > 9 else 3
    R, S_, sd, pd = sch.pop("_geom", (3, 3, 1, 1))     # optional filter / stride / pad in the JSON
    d = xtc.conv2d_desc(B, H, W, C, F, R, S_, sd, pd, ind, outd); sa, sb = (B, H, W, C), (R, S_, C, F)
Mg, Ng, Kg = xtc.gemm_view(d)
x = torch.empty(sa, dtype=T[ind], device="cuda"); w = torch.empty(sb, dtype=T[ind], device="cuda")
y = torch.empty((Mg, Ng), dtype=T[outd], device="cuda")
st = torch.cuda.current_stream().cuda_stream
xtc.xtc_fill(x.data_ptr(), x.numel(), xtc.DTYPES[ind], 1, 0, 0, st); xtc.xtc_fill(w.data_ptr(), w.numel(), xtc.DTYPES[ind], 2, 0, 0, st)
# RUN_ONE_WARM=n: n untraced launches first (clocks ramp up), the XTC_TRACE op is created afterwards
warm = int(os.environ.get("RUN_ONE_WARM", "0"))
if warm:
    tr = os.environ.pop("XTC_TRACE", None)
    op0 = xtc.Op(d).apply(xtc.schedule(**sch))
    for _ in range(warm):
        op0.run(x, w, y)
    torch.cuda.synchronize()
    if tr:
        os.environ["XTC_TRACE"] = tr
op = xtc.Op(d).apply(xtc.schedule(**sch))
for _ in range(reps):
    op.run(x, w, y)
torch.cuda.synchronize()
print("ok", a[0], Mg, Ng, Kg)
