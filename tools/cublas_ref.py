import torch
a = torch.randn(8192, 8192, dtype=torch.bfloat16, device="cuda"); b = torch.randn(8192, 8192, dtype=torch.bfloat16, device="cuda")
for _ in range(3): c = torch.matmul(a, b)
torch.cuda.synchronize()
