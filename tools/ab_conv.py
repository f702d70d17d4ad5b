#!/usr/bin/env python3
"""Time a few memory-bound convs (CUDA events, L2-cold inputs) with whichever
paper_1910_00932_b200 is first on sys.path (A/B of two builds on one box)."""
import sys
import torch
import paper_1910_00932_b200 as pkg
from paper_1910_00932_b200 import conv

dev = torch.device("cuda", 0)
B = 64


def timeit(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(True), torch.cuda.Event(True)
        a.record(); fn(); b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    ts.sort()
    return ts[len(ts) // 2]


x64 = torch.randn(B, 8, 56, 56, 64, device=dev).bfloat16()
r256 = torch.randn(B, 8, 56, 56, 256, device=dev).bfloat16()
y256 = torch.empty_like(r256)
w = (torch.randn(256, 64, device=dev) / 8).bfloat16()
bias = torch.zeros(256, device=dev)
res = {
    "proj64_256": timeit(lambda: conv.conv1x1_fwd(x64, w, bias, out=y256)),
    "proj_nobias": timeit(lambda: conv.conv1x1_fwd(x64, w, None, out=y256)),
    "c3res64_256": timeit(lambda: conv.conv1x1_fwd(x64, w, bias, residual=r256, relu=True, out=y256)),
}
x128 = torch.randn(B, 8, 28, 28, 128, device=dev).bfloat16()
r512 = torch.randn(B, 8, 28, 28, 512, device=dev).bfloat16()
y512 = torch.empty_like(r512)
w2 = (torch.randn(512, 128, device=dev) / 8).bfloat16()
b2 = torch.zeros(512, device=dev)
res["c3res128_512"] = timeit(lambda: conv.conv1x1_fwd(x128, w2, b2, residual=r512, relu=True, out=y512))
print(pkg.__file__, {k: round(v, 1) for k, v in res.items()})

if len(sys.argv) > 1 and sys.argv[1] == "proj-only":
    pass
