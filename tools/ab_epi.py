#!/usr/bin/env python3
"""Time the res2-shaped memory-bound GEMMs (CUDA events, median of 10) with
whichever paper_1910_00932_b200 is first on sys.path — run once per
tools/build_variant.sh variant to A/B epilogue experiments on one box."""
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
x256 = torch.randn(B, 8, 56, 56, 256, device=dev).bfloat16()
y256 = torch.empty_like(x256)
y64 = torch.empty_like(x64)
w = (torch.randn(256, 64, device=dev) / 8).bfloat16()
w1 = (torch.randn(64, 256, device=dev) / 16).bfloat16()
wt = (torch.randn(256, 1, 1, 64, device=dev) / 8).bfloat16()
bias = torch.zeros(256, device=dev)
b64 = torch.zeros(64, device=dev)
res = {
    "proj64_256": timeit(lambda: conv.conv1x1_fwd(x64, w, bias, out=y256)),
    "c3res64_256": timeit(lambda: conv.conv1x1_fwd(x64, w, bias, residual=x256, relu=True, out=y256)),
    "dgrad_c1_shift": timeit(lambda: conv.conv_dgrad(x64, wt, x256.shape, fold=(32, 32), out=y256)),
    "c1fwd256_64": timeit(lambda: conv.conv1x1_fwd(x256, w1, b64, fold=(32, 32), relu=True, out=y64)),
}
print(pkg.__file__.split("/")[-3], {k: round(v, 1) for k, v in res.items()})
