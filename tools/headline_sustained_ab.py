"""Headline default A/B under the bench protocol: blocks of 100 back-to-back launches (as bench.py's
timed region), the two candidate defaults interleaved, 1 s idle between blocks; TFLOP/s per block."""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2512_16512_b200 as xtc
import bench
n = 8192
st = torch.cuda.current_stream().cuda_stream
a = torch.empty((n, n), dtype=torch.bfloat16, device="cuda")
b = torch.empty((n, n), dtype=torch.bfloat16, device="cuda")
c = torch.empty((n, n), dtype=torch.bfloat16, device="cuda")
xtc.xtc_fill(a.data_ptr(), a.numel(), xtc.XTC_BF16, 1, 0, 0, st)
xtc.xtc_fill(b.data_ptr(), b.numel(), xtc.XTC_BF16, 2, 0, 0, st)
ops = {"pair512_ms2": xtc.Op(xtc.matmul_desc(n, n, n)).apply(xtc.schedule(**bench.HEADLINE_SCHEDULE)),
       "pair512_ms2_4stage_plain_epilogue": xtc.Op(xtc.matmul_desc(n, n, n)).apply(
           xtc.schedule(**dict(bench.HEADLINE_SCHEDULE, stages=4))),
       "pair256": xtc.Op(xtc.matmul_desc(n, n, n)).apply(xtc.schedule(**bench.PAIR256_SCHEDULE))}
res = {k: [] for k in ops}
for rnd in range(4):
    for name, op in (ops.items() if rnd % 2 == 0 else reversed(list(ops.items()))):
        for _ in range(10):
            op.run(a, b, c)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(100):
            op.run(a, b, c)
        e1.record()
        torch.cuda.synchronize()
        res[name].append(round(2 * n ** 3 / (e0.elapsed_time(e1) / 100 * 1e-3) / 1e12, 1))
        time.sleep(1.0)
print(json.dumps(res))
