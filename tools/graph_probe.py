#!/usr/bin/env python3
"""Does one train step capture into a CUDA graph, and how much faster does the
replay run than eager launches?  (Experiment; 1 GPU, batch 64.)"""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1910_00932_b200.network import TSMNet  # noqa: E402

dev = torch.device("cuda", 0)
net = TSMNet(batch=64, device=dev).init_random(0)
x = torch.randn(64, 8, 3, 224, 224, device=dev)
for _ in range(3):
    net.train_step(x, lr=1e-13)
torch.cuda.synchronize()


def timeit(fn, n=10):
    a, b = torch.cuda.Event(True), torch.cuda.Event(True)
    a.record()
    for _ in range(n):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n


eager = timeit(lambda: net.train_step(x, lr=1e-13))
s = torch.cuda.Stream(dev)
s.wait_stream(torch.cuda.current_stream(dev))
g = torch.cuda.CUDAGraph()
try:
    with torch.cuda.stream(s):
        net.train_step(x, lr=1e-13)  # warm on the capture stream
    torch.cuda.synchronize()
    with torch.cuda.graph(g, stream=s):
        net.train_step(x, lr=1e-13)
    torch.cuda.synchronize()
    graph = timeit(lambda: g.replay())
    print(f"eager {eager:.3f} ms/step, graph replay {graph:.3f} ms/step")
except Exception as e:  # noqa: BLE001
    print(f"eager {eager:.3f} ms/step; capture failed: {e}")
