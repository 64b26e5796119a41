"""cuDNN conv2d (channels_last bf16, benchmark mode) at one BASELINE layer, a few launches (for ncu).
Usage: cudnn_conv_one.py n h c"""
import sys
import torch
import torch.nn.functional as F
n, h, c = map(int, sys.argv[1:4])
torch.backends.cudnn.benchmark = True
x = torch.randn(n, c, h, h, device="cuda", dtype=torch.bfloat16).to(memory_format=torch.channels_last)
w = torch.randn(c, c, 3, 3, device="cuda", dtype=torch.bfloat16).to(memory_format=torch.channels_last)
for _ in range(20):
    F.conv2d(x, w, padding=1)
torch.cuda.synchronize()
print("ok")
