#!/usr/bin/env python3
"""A/B of the north-star kernel (fused shift + 1x1 conv, res2 conv1:
C=256 -> 64, F=32, 64 clips, 56x56, T=8) and two neighbouring res2 GEMMs,
timed like bench.py's roofline leg (CUDA events, L2 flushed between
launches), with whichever paper_1910_00932_b200 is first on sys.path.

    PYTHONPATH=_ab/<variant> python tools/ab_conv1.py <label>"""
import statistics
import sys

import torch
import paper_1910_00932_b200 as pkg
from paper_1910_00932_b200 import conv

dev = torch.device("cuda", 0)
n, t, h, w = 64, 8, 56, 56
m = n * t * h * w
flush = torch.empty(64 * 1024 * 1024, device=dev)


def timeit(fn, reps=15):
    for _ in range(3):
        fn()
    ts = []
    for _ in range(reps):
        flush.fill_(1.0)
        a, b = torch.cuda.Event(True), torch.cuda.Event(True)
        a.record(); fn(); b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    return statistics.median(ts)


x256 = torch.randn(n, t, h, w, 256, device=dev).bfloat16()
x64 = torch.randn(n, t, h, w, 64, device=dev).bfloat16()
w1 = (torch.randn(64, 256, device=dev) / 16).bfloat16()
w3 = (torch.randn(256, 64, device=dev) / 8).bfloat16()
b64, b256 = torch.zeros(64, device=dev), torch.zeros(256, device=dev)
y64 = torch.empty_like(x64)
y256 = torch.empty_like(x256)
cases = {
    "conv1 shift C256->64": (lambda: conv.conv1x1_fwd(x256, w1, b64, fold=(32, 32), relu=True, out=y64),
                             2 * (m * 256 + m * 64)),
    "conv3+res C64->256": (lambda: conv.conv1x1_fwd(x64, w3, b256, relu=True, residual=x256, out=y256),
                           2 * (m * 64 + 2 * m * 256)),
    "proj C64->256": (lambda: conv.conv1x1_fwd(x64, w3, b256, out=y256), 2 * (m * 64 + m * 256)),
}
label = sys.argv[1] if len(sys.argv) > 1 else pkg.__file__
for name, (fn, nbytes) in cases.items():
    us = timeit(fn)
    print(f"{label:8s} {name:22s} {us:8.1f} us  {nbytes / us / 1e3:7.0f} GB/s", flush=True)
