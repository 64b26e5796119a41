"""cuDNN (torch.nn.functional.conv2d, channels_last bf16) time for the BASELINE conv
configs -- a library reference point for the implicit-GEMM kernel, L2 flushed per rep."""
import torch, json
import torch.nn.functional as F

def t_conv(n, h, c, f, reps=50):
    x = torch.randn(n, c, h, h, device="cuda", dtype=torch.bfloat16).to(memory_format=torch.channels_last)
    w = torch.randn(f, c, 3, 3, device="cuda", dtype=torch.bfloat16).to(memory_format=torch.channels_last)
    flush = torch.empty(512 * 1024 * 1024 // 4, device="cuda", dtype=torch.float32)
    for _ in range(5):
        F.conv2d(x, w, padding=1)
    ts = []
    for _ in range(reps):
        flush.sum()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); F.conv2d(x, w, padding=1); e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    ts.sort()
    med = ts[len(ts) // 2]
    fl = 2 * n * h * h * f * 9 * c
    return {"t_med_us": round(med, 2), "tflops": round(fl / med * 1e-6, 1)}

torch.backends.cudnn.benchmark = True
out = {}
for name, (h, c) in {"L56": (56, 64), "L14": (14, 256)}.items():
    for n in (1, 8, 32):
        out[f"{name}_n{n}"] = t_conv(n, h, c, c)
print(json.dumps(out, indent=1))
