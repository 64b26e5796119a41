"""torch.matmul (cuBLAS) at n^3 bf16, a few launches (for ncu captures).  Usage: cublas_small_one.py n"""
import sys
import torch
n = int(sys.argv[1])
a = torch.randn(n, n, dtype=torch.bfloat16, device="cuda")
b = torch.randn(n, n, dtype=torch.bfloat16, device="cuda")
c = torch.empty(n, n, dtype=torch.bfloat16, device="cuda")
for _ in range(3):
    torch.matmul(a, b, out=c)
torch.cuda.synchronize()
print("ok")
