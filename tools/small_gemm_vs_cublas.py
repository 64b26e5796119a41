"""512^3 / 1024^3 bf16 (BASELINE config 2) under one protocol for xtc and cuBLAS (torch.matmul):
L2 flushed by a 2xL2 read before every rep, each rep between CUDA events on the launching stream;
median and mean of 30 reps, interleaved rounds.  Also empty-kernel and torch.add floors."""
import os, sys, json, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2512_16512_b200 as xtc
from paper_2512_16512_b200.bench_extras import MATMUL_SCHEDS

dev = torch.device("cuda", 0)
st = torch.cuda.current_stream()
flush = torch.empty(2 * 126 * 2**20 // 4, dtype=torch.float32, device=dev).uniform_()
sink = torch.empty((), dtype=torch.float32, device=dev)


def timeit(fn, reps=30):
    ts = []
    for _ in range(3):
        fn()
    for _ in range(reps):
        sink.copy_(flush.sum())
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        fn()
        e1.record(st)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    return round(statistics.median(ts), 2), round(statistics.mean(ts), 2)


res = {}
for n in (512, 1024):
    a = torch.empty((n, n), dtype=torch.bfloat16, device=dev)
    b = torch.empty((n, n), dtype=torch.bfloat16, device=dev)
    c = torch.empty((n, n), dtype=torch.bfloat16, device=dev)
    xtc.xtc_fill(a.data_ptr(), a.numel(), xtc.XTC_BF16, 1, 0, 0, st.cuda_stream)
    xtc.xtc_fill(b.data_ptr(), b.numel(), xtc.XTC_BF16, 2, 0, 0, st.cuda_stream)
    ops = []
    TC = dict(engine=1, tile_m=128, tile_k=64, swizzle=128, buffer_c=1)
    extra = [dict(TC, tile_n=64, stages=8, cluster_n=2), dict(TC, tile_n=64, stages=8, cluster_n=4),
             dict(TC, tile_n=64, stages=8, cluster_n=2, acc_buffers=2, persistent=1),
             dict(TC, tile_n=64, stages=8, cluster_n=4, pack_warps=2),
             dict(TC, tile_n=128, stages=6, cluster_n=2), dict(TC, tile_n=64, tile_k=128, stages=4, cluster_n=4)]
    for i, s in enumerate(list(MATMUL_SCHEDS[n]) + extra):
        try:
            ops.append((f"xtc{i}", xtc.Op(xtc.matmul_desc(n, n, n)).apply(xtc.schedule(**s))))
        except xtc.XtcError:
            pass
    for rnd in range(3):
        r = res.setdefault(str(n), {})
        r.setdefault("cublas", []).append(timeit(lambda: torch.matmul(a, b, out=c)))
        for name, op in ops:
            r.setdefault(name, []).append(timeit(lambda: op.run(a, b, c)))
small = torch.empty(16, device=dev)
res["floor_torch_add_16"] = [timeit(lambda: small.add_(1.0)) for _ in range(2)]
print(json.dumps(res, indent=1))
