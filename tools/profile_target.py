#!/usr/bin/env python3
"""Small, deterministic launch sequences for ncu (run it plain first, then
under ncu; never multi-rank).

    python tools/profile_target.py step   [--batch 64]  # 2 warm-up steps + 1 train step
    python tools/profile_target.py conv1  [--batch 64]  # fused shift + 1x1 conv (res2 conv1)
    python tools/profile_target.py shift                # temporal shift fwd on (8,8,256,56,56) f32
"""
import argparse
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import os  # noqa: E402
if os.environ.get("TSM_PKG_ROOT"):  # profile another build of the package
    sys.path.insert(0, os.environ["TSM_PKG_ROOT"])


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("what", choices=["step", "conv1", "shift", "wgrad5", "wgrad2", "conv3x3", "conv3res", "wgrad3", "wgrad3c1", "subpix", "fused", "wgrad4c3", "conv3res4", "conv1r5", "fwd", "wgrad4c2", "halo128"])
    ap.add_argument("--batch", type=int, default=64)
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    if a.what == "step":
        from paper_1910_00932_b200.network import TSMNet
        net = TSMNet(batch=a.batch, device=dev).init_random(0)
        x = torch.randn(a.batch, 8, 3, 224, 224, device=dev)
        for _ in range(2):
            net.train_step(x, lr=1e-13)
        torch.cuda.synchronize()
        # exactly one step inside the profiler range (ncu --profile-from-start off)
        torch.cuda.profiler.start()
        net.train_step(x, lr=1e-13)
        torch.cuda.synchronize()
        torch.cuda.profiler.stop()
    elif a.what == "conv1":
        from paper_1910_00932_b200 import conv
        x = torch.randn(a.batch, 8, 56, 56, 256, device=dev).bfloat16()
        w = (torch.randn(64, 256, device=dev) / 16).bfloat16()
        b = torch.zeros(64, device=dev)
        y = torch.empty(a.batch, 8, 56, 56, 64, device=dev, dtype=torch.bfloat16)
        for _ in range(4):
            conv.conv1x1_fwd(x, w, b, fold=(32, 32), relu=True, out=y)
    elif a.what in ("wgrad3", "wgrad3c1"):
        from paper_1910_00932_b200 import conv
        if a.what == "wgrad3":   # res3 conv2: 128 -> 128, 3x3, 28x28
            x = torch.randn(a.batch, 8, 28, 28, 128, device=dev).bfloat16()
            dy = torch.randn(a.batch, 8, 28, 28, 128, device=dev).bfloat16()
            k = 3
        else:                    # res3 conv1: 512 -> 128, 1x1, 28x28
            x = torch.randn(a.batch, 8, 28, 28, 512, device=dev).bfloat16()
            dy = torch.randn(a.batch, 8, 28, 28, 128, device=dev).bfloat16()
            k = 1
        for _ in range(4):
            conv.conv_wgrad(x, dy, k=k, bias_grad=True)
    elif a.what in ("wgrad5", "wgrad2"):
        from paper_1910_00932_b200 import conv
        if a.what == "wgrad5":   # res5 conv3: 512 -> 2048, 1x1, 7x7
            x = torch.randn(a.batch, 8, 7, 7, 512, device=dev).bfloat16()
            dy = torch.randn(a.batch, 8, 7, 7, 2048, device=dev).bfloat16()
            k = 1
        else:                    # res2 conv2: 64 -> 64, 3x3, 56x56
            x = torch.randn(a.batch, 8, 56, 56, 64, device=dev).bfloat16()
            dy = torch.randn(a.batch, 8, 56, 56, 64, device=dev).bfloat16()
            k = 3
        for _ in range(4):
            conv.conv_wgrad(x, dy, k=k)
    elif a.what == "wgrad4c2":   # res4 conv2 weight gradient: 3x3 256 -> 256 @14 (CTA pair)
        from paper_1910_00932_b200 import conv
        x = torch.randn(a.batch, 8, 14, 14, 256, device=dev).bfloat16()
        dy = torch.randn(a.batch, 8, 14, 14, 256, device=dev).bfloat16()
        for _ in range(4):
            conv.conv_wgrad(x, dy, k=3)
    elif a.what == "wgrad4c3":   # res4 conv3 weight gradient: 256 -> 1024, 1x1, 14x14 (+ db)
        from paper_1910_00932_b200 import conv
        x = torch.randn(a.batch, 8, 14, 14, 256, device=dev).bfloat16()
        dy = torch.randn(a.batch, 8, 14, 14, 1024, device=dev).bfloat16()
        for _ in range(4):
            conv.conv_wgrad(x, dy, k=1, bias_grad=True)
    elif a.what == "fused":      # res2 identity unit forward, fused (TSM_FUSED_BLOCK=1)
        os.environ["TSM_FUSED_BLOCK"] = "1"
        from paper_1910_00932_b200.block import Bottleneck
        blk = Bottleneck(256, 256, 1, device=dev)
        g = torch.Generator(device=dev).manual_seed(0)
        for k, s in blk.shapes().items():
            blk.params[k] = torch.randn(s, device=dev, generator=g) * (0.05 if k[0] == "w" else 0.1)
        x = torch.randn(a.batch, 8, 56, 56, 256, device=dev).bfloat16()
        for _ in range(4):
            blk.forward(x)
    elif a.what == "conv3res":   # res2 conv3 forward: 64 -> 256, + residual, relu
        from paper_1910_00932_b200 import conv
        x = torch.randn(a.batch, 8, 56, 56, 64, device=dev).bfloat16()
        r = torch.randn(a.batch, 8, 56, 56, 256, device=dev).bfloat16()
        w = (torch.randn(256, 64, device=dev) / 8).bfloat16()
        b = torch.zeros(256, device=dev)
        y = torch.empty_like(r)
        for _ in range(4):
            conv.conv1x1_fwd(x, w, b, residual=r, relu=True, out=y)
    elif a.what == "fwd":        # network forward (stem, pool, all units, head)
        from paper_1910_00932_b200.network import TSMNet
        net = TSMNet(batch=a.batch, device=dev).init_random(0)
        x = torch.randn(a.batch, 8, 3, 224, 224, device=dev)
        for _ in range(2):
            net.forward(x)
        torch.cuda.synchronize()
    elif a.what == "conv3res4":  # res4 conv3 forward: 256 -> 1024 @14, + residual, relu
        from paper_1910_00932_b200 import conv
        x = torch.randn(a.batch, 8, 14, 14, 256, device=dev).bfloat16()
        r = torch.randn(a.batch, 8, 14, 14, 1024, device=dev).bfloat16()
        w = (torch.randn(1024, 256, device=dev) / 16).bfloat16()
        b = torch.zeros(1024, device=dev)
        y = torch.empty_like(r)
        for _ in range(4):
            conv.conv1x1_fwd(x, w, b, residual=r, relu=True, out=y)
    elif a.what == "conv1r5":    # res5 fused shift + conv1: 2048 -> 512 @7, fold 256
        from paper_1910_00932_b200 import conv
        x = torch.randn(a.batch, 8, 7, 7, 2048, device=dev).bfloat16()
        w = (torch.randn(512, 2048, device=dev) / 45).bfloat16()
        b = torch.zeros(512, device=dev)
        y = torch.empty(a.batch, 8, 7, 7, 512, device=dev, dtype=torch.bfloat16)
        for _ in range(4):
            conv.conv1x1_fwd(x, w, b, fold=(256, 256), relu=True, out=y)
    elif a.what == "subpix":     # res3 first-unit conv2 dgrad: 3x3 / s2, 128 -> 128, 4 classes
        from paper_1910_00932_b200 import conv
        dy = torch.randn(a.batch, 8, 28, 28, 128, device=dev).bfloat16()
        wt = (torch.randn(128, 3, 3, 128, device=dev) / 32).bfloat16()
        dx = torch.empty(a.batch, 8, 56, 56, 128, device=dev, dtype=torch.bfloat16)
        for _ in range(2):
            conv.conv_dgrad(dy, wt, dx.shape, k=3, stride=2, out=dx)
    elif a.what == "halo128":    # res3 conv2 forward: 3x3 128 -> 128 @28 (halo, CTA pairs)
        from paper_1910_00932_b200 import conv
        x = torch.randn(a.batch, 8, 28, 28, 128, device=dev).bfloat16()
        w = (torch.randn(128, 1152, device=dev) / 34).bfloat16()
        b = torch.zeros(128, device=dev)
        for _ in range(4):
            conv.conv_fwd(x, w, b, k=3, relu=True)
    elif a.what == "conv3x3":    # res2 conv2 forward
        from paper_1910_00932_b200 import conv
        x = torch.randn(a.batch, 8, 56, 56, 64, device=dev).bfloat16()
        w = (torch.randn(64, 576, device=dev) / 24).bfloat16()
        b = torch.zeros(64, device=dev)
        for _ in range(4):
            conv.conv_fwd(x, w, b, k=3, relu=True)
    else:
        import paper_1910_00932_b200 as tsm
        x = torch.randn(8, 8, 256, 56, 56, device=dev)
        y = torch.empty_like(x)
        for _ in range(4):
            tsm.temporal_shift(x, tsm.ShiftConfig.fold_div(8), out=y)
    torch.cuda.synchronize()
    print("ok")


if __name__ == "__main__":
    main()
