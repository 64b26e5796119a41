import torch, time
N = 128 * 1024 * 1024
ha = torch.empty(N, dtype=torch.uint8).pin_memory(); hb = torch.empty(N, dtype=torch.uint8).pin_memory()
hc = torch.empty(N, dtype=torch.uint8).pin_memory()
da = torch.empty(N, dtype=torch.uint8, device="cuda"); db = torch.empty_like(da); dc = torch.empty_like(da)
s1, s2, s3 = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
def t(fn, reps=5):
    fn(); torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    for _ in range(reps): fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps
def one():
    with torch.cuda.stream(s1):
        da.copy_(ha, non_blocking=True); db.copy_(hb, non_blocking=True)
def two():
    with torch.cuda.stream(s1): da.copy_(ha, non_blocking=True)
    with torch.cuda.stream(s2): db.copy_(hb, non_blocking=True)
def dup():
    with torch.cuda.stream(s1):
        da.copy_(ha, non_blocking=True); db.copy_(hb, non_blocking=True)
    with torch.cuda.stream(s3): hc.copy_(dc, non_blocking=True)
for name, fn, nbytes in (("H2D 256MB 1 stream", one, 2 * N), ("H2D 256MB 2 streams", two, 2 * N), ("H2D 256MB + D2H 128MB", dup, 2 * N)):
    dt = t(fn)
    print(f"{name}: {dt*1e3:.2f} ms  {nbytes/dt/1e9:.1f} GB/s (H2D)", flush=True)
