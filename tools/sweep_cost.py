"""Decompose xtc_sweep's per-candidate cost (1024^3 bf16, the bench's candidate list): PYTHONPATH=. python tools/sweep_cost.py"""
import time
import torch
import paper_2512_16512_b200 as xtc
from paper_2512_16512_b200.sweep import run_sweep
_, samples, mine, todo, scheds, op, (a, b, c), cfg, sp, _ = run_sweep(1024, 1024, 1024, 512, seed=0, world=1, rank=0,
                                                                      device=0, peak_tflops=1669.1)
for v, w, r in ((1, 2, 10), (0, 0, 1), (1, 0, 1), (0, 0, 10), (0, 2, 10), (1, 2, 10)):
    mc = xtc.measure_cfg(warmup=w, repeats=r, validate=v, reuse_reference=1, tol=5e-3)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    op.sweep(scheds, a, b, c, mc, stream=sp)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(f"validate {v} warmup {w} repeats {r}: {dt * 1e3:.1f} ms for {len(scheds)} -> {dt / len(scheds) * 1e6:.1f} us per candidate",
          flush=True)
