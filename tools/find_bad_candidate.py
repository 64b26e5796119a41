"""Run the schedule-invariance candidates of test_schedule_invariance_tcgen05_sampled one by one
(sync after each), printing the index first: the last index printed before a failure is the culprit."""
import sys
import torch
import paper_2512_16512_b200 as xtc
from paper_2512_16512_b200.strategy import GpuStrategy
desc = xtc.matmul_desc(512, 512, 512, "bf16", "bf16")
st = GpuStrategy(desc, exact_divisors=False)
cands = [st.generate(s) for s in st.sample(128, seed=11)]
extra = []
for i, c in enumerate(cands[:32]):
    d = c.as_dict(); d["pack_warps"] = 1 + i % 3; extra.append(xtc.schedule(**d))
allc = cands + extra
a = torch.ones((512, 512), dtype=torch.bfloat16, device="cuda"); b = torch.ones_like(a)
c = torch.empty_like(a)
op = xtc.Op(desc)
start = int(sys.argv[1]) if len(sys.argv) > 1 else 0
for i, s in enumerate(allc[start:], start):
    print(i, s.as_dict(), flush=True)
    op.apply(s)
    op.run(a, b, c)
    torch.cuda.synchronize()
print("all ok")
