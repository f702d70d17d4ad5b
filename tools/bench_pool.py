#!/usr/bin/env python3
"""Max pool forward / backward at the TSM-R50 stem shape (64 clips x 8
frames, 112 x 112 x 64 bf16 -> 56 x 56), CUDA events, median of 20 launches;
HBM GB/s of the algorithmic bytes (x + y + argmax; gy + argmax + gx).

    TSM_POOL_R=1|2|3 TSM_POOL_BR=2|4|8 python tools/bench_pool.py"""
import json
import os
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1910_00932_b200 import conv  # noqa: E402


def time_us(fn, reps=20, warm=5):
    for _ in range(warm):
        fn()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(reps)]
    for a, b in ev:
        a.record()
        fn()
        b.record()
    torch.cuda.synchronize()
    t = sorted(a.elapsed_time(b) for a, b in ev)
    return 1e3 * t[len(t) // 2]


def main():
    x = torch.randn(64, 8, 112, 112, 64, device="cuda").bfloat16()
    y, arg = conv.maxpool_fwd(x)
    gy = torch.randn_like(y.float()).bfloat16()
    fwd = time_us(lambda: conv.maxpool_fwd(x))
    bwd = time_us(lambda: conv.maxpool_bwd(gy, arg, x.shape))
    nb_f = x.numel() * 2 + y.numel() * 3
    nb_b = gy.numel() * 3 + x.numel() * 2
    print(json.dumps({"R": os.environ.get("TSM_POOL_R", "2"), "BR": os.environ.get("TSM_POOL_BR", "4"),
                      "fwd_us": round(fwd, 1), "fwd_GBps": round(nb_f / fwd / 1e3, 1),
                      "bwd_us": round(bwd, 1), "bwd_GBps": round(nb_b / bwd / 1e3, 1)}))


if __name__ == "__main__":
    main()
