#!/usr/bin/env python3
"""One proj conv (64 -> 256, 56x56, batch 64) for ncu A/B of two builds."""
import torch
from paper_1910_00932_b200 import conv
dev = torch.device("cuda", 0)
x64 = torch.randn(64, 8, 56, 56, 64, device=dev).bfloat16()
y = torch.empty(64, 8, 56, 56, 256, device=dev).bfloat16()
w = (torch.randn(256, 64, device=dev) / 8).bfloat16()
b = torch.zeros(256, device=dev)
for _ in range(3):
    conv.conv1x1_fwd(x64, w, b, out=y)
torch.cuda.synchronize()
print("ok")
