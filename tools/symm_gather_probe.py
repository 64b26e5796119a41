"""GPU probe of the fused all-gather (xtc_run_gather) plumbing at world size 1 under torchrun:
the symmetric-memory rendezvous + barrier bench.py --gather fused uses, and the epilogue cost of
storing every tile to W destinations (here W local buffers) on the 8192^3 headline GEMM."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import torch.distributed as dist
import paper_2512_16512_b200 as xtc
from paper_2512_16512_b200.parallel import SymmetricOutput
from bench import HEADLINE_SCHEDULE

dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
dist.init_process_group("nccl", device_id=dev)
out = {}
st = torch.cuda.current_stream().cuda_stream
for Ms in (8192, 1024):
    M = N = K = 8192
    a = torch.empty((Ms, K), dtype=torch.bfloat16, device=dev)
    b = torch.empty((K, N), dtype=torch.bfloat16, device=dev)
    xtc.xtc_fill(a.data_ptr(), a.numel(), xtc.XTC_BF16, 1, 0, 0, st)
    xtc.xtc_fill(b.data_ptr(), b.numel(), xtc.XTC_BF16, 2, 0, 0, st)
    op = xtc.Op(xtc.matmul_desc(Ms, N, K)).apply(xtc.schedule(**HEADLINE_SCHEDULE))
    c = torch.empty((Ms, N), dtype=torch.bfloat16, device=dev)
    sym = SymmetricOutput((M, N), torch.bfloat16, dev)
    res = {"symm_dests": len(sym.dests)}
    op.run(a, b, c)
    op.run_gather(a, b, sym.dests, 0, M)
    sym.barrier()
    torch.cuda.synchronize()
    res["symm_equal_local"] = bool(torch.equal(sym.tensor[:Ms], c))
    extra = [torch.empty((M, N), dtype=torch.bfloat16, device=dev) for _ in range(7)]

    def timeit(fn, reps=20):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps * 1e3

    for rnd in range(2):
        res[f"run_us_{rnd}"] = timeit(lambda: op.run(a, b, c))
        res[f"gather1_symm_us_{rnd}"] = timeit(lambda: (op.run_gather(a, b, sym.dests, 0, M), sym.barrier()))
        ptrs8 = [sym.dests[0]] + [e.data_ptr() for e in extra]
        res[f"gather8_local_us_{rnd}"] = timeit(lambda: op.run_gather(a, b, ptrs8, 0, M))
    torch.cuda.synchronize()
    res["gather8_all_equal"] = all(bool(torch.equal(e[:Ms], c)) for e in extra)
    out[f"M_shard_{Ms}"] = res
print(json.dumps(out))
dist.destroy_process_group()
