"""Small-GEMM schedule search on the current build: the legal-set sweep (GpuStrategy, 4096 seeded
candidates, warm L2) for 512^3 / 1024^3 bf16, then the top 16 re-measured with the bench protocol
(L2 flushed, 20 reps, validated).  PYTHONPATH=. python tools/small_gemm_search.py"""
import json
import torch
import paper_2512_16512_b200 as xtc
from paper_2512_16512_b200.strategy import GpuStrategy
from paper_2512_16512_b200.bench_extras import _best, MATMUL_SCHEDS

dev = torch.device("cuda", 0)
for n in (512, 1024):
    desc = xtc.matmul_desc(n, n, n, "bf16", "bf16")
    st = GpuStrategy(desc)
    cands = [st.generate(s) for s in st.sample(4096, seed=3)]
    a = torch.empty((n, n), dtype=torch.bfloat16, device=dev); b = torch.empty_like(a); c = torch.empty_like(a)
    s_ = torch.cuda.current_stream().cuda_stream
    xtc.xtc_fill(a.data_ptr(), a.numel(), xtc.XTC_BF16, 5, 0, 0, s_); xtc.xtc_fill(b.data_ptr(), b.numel(), xtc.XTC_BF16, 6, 0, 0, s_)
    op = xtc.Op(desc)
    recs = op.sweep(cands, a, b, c, xtc.measure_cfg(warmup=2, repeats=10, flush_l2=1, validate=1, reuse_reference=1))
    ok = sorted([(r.t_med_ns, i) for i, r in enumerate(recs) if r.status == 0 and r.valid == 1])
    seen, top = set(), []
    for t, i in ok:
        d = cands[i].as_dict()
        key = json.dumps(d, sort_keys=True)
        if key in seen:
            continue
        seen.add(key); top.append(d)
        if len(top) == 16:
            break
    top = [{k: v for k, v in d.items() if v} for d in top]
    r = _best(xtc, torch, dev, desc, top + MATMUL_SCHEDS[n], [(n, n), (n, n)], 1638.9)
    print(json.dumps({"n": n, "sweep_best_us": ok[0][0] / 1e3, "best_us": r["t_med_us"], "best": r["schedule"],
                      "tried": [t.get("t_med_us") for t in r["tried"]]}), flush=True)
    for d, t in zip(top, r["tried"]):
        print("   ", t.get("t_med_us"), d)
