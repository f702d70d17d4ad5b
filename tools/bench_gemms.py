#!/usr/bin/env python3
"""Per-kernel timing of the compute-bound res3-res5 convolutions of the
TSM-R50 step at 64 clips (CUDA events on the launching stream, 5 warm-up +
20 timed launches, inputs > L2 except the res5 weights).

    TSM_PAIR=0|1 python tools/bench_gemms.py [--json out.json]

TSM_PAIR selects the single-CTA (0) or CTA-pair (cta_group::2, 1) tcgen05
GEMM for the eligible shapes (conv_ops.cu use_pair); run both on one box for
an A/B.  Prints per case: µs, TFLOP/s and the fraction of the burst bf16
peak (MEASURED_PEAKS.json), plus HBM GB/s of the algorithmic bytes."""
from __future__ import annotations

import argparse
import json
import os
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from paper_1910_00932_b200 import conv  # noqa: E402


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    d = json.loads(p.read_text()) if p.exists() else {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}
    return d["hbm_gbs"], d["bf16_tflops"]


def time_us(fn, reps=20, warm=5):
    s = torch.cuda.current_stream()
    for _ in range(warm):
        fn()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(reps)]
    for a, b in ev:
        a.record(s)
        fn()
        b.record(s)
    torch.cuda.synchronize()
    t = sorted(a.elapsed_time(b) for a, b in ev)
    return 1e3 * t[len(t) // 2]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--json")
    ap.add_argument("--clips", type=int, default=64)
    ap.add_argument("--only", default="", help="substring filter on the case names")
    a = ap.parse_args()
    hbm, tf = peaks()
    dev = torch.device("cuda")
    N, T = a.clips, 8
    torch.manual_seed(0)
    rows = []

    def report(name, us, flops, nbytes):
        if a.only and a.only not in name:
            return
        r = {"case": name, "us": round(us, 1), "TFLOPs": round(flops / us / 1e6, 1),
             "frac_burst": round(flops / us / 1e6 / tf, 3),
             "GBps": round(nbytes / us / 1e3, 1), "pair": os.environ.get("TSM_PAIR", "1")}
        rows.append(r)
        print(json.dumps(r), flush=True)

    def bf(*shape, scale=1.0):
        return (torch.randn(*shape, device=dev) * scale).bfloat16()

    # fused shift + 1x1 conv1 (north-star b) at res4 / res5
    for h, cin, cout in ((28, 512, 128), (14, 1024, 256), (7, 2048, 512)):
        x = bf(N, T, h, h, cin)
        w = bf(cout, 1, 1, cin, scale=cin ** -0.5)
        b = torch.zeros(cout, device=dev)
        y = torch.empty(N, T, h, h, cout, device=dev, dtype=torch.bfloat16)
        f = cin // 8
        us = time_us(lambda: conv.conv_fwd(x, w, b, fold=(f, f), relu=True, out=y))
        m = N * T * h * h
        report(f"fwd shift+conv1 {cin}->{cout} @{h}", us, 2 * m * cin * cout,
               2 * (m * cin + m * cout + cin * cout))
        del x, y
    # 3x3 forward at res2 (halo) and res3 - res5
    for h, c in ((56, 64), (28, 128), (14, 256), (7, 512)):
        x = bf(N, T, h, h, c)
        w = bf(c, 3, 3, c, scale=(9 * c) ** -0.5)
        b = torch.zeros(c, device=dev)
        y = torch.empty(N, T, h, h, c, device=dev, dtype=torch.bfloat16)
        us = time_us(lambda: conv.conv_fwd(x, w, b, k=3, relu=True, out=y))
        m = N * T * h * h
        report(f"fwd conv2 3x3 {c} @{h}", us, 2 * m * 9 * c * c, 2 * (2 * m * c + 9 * c * c))
        # stride-1 3x3 dgrad (tap-flipped weights) with a ReLU mask
        wf, wd = conv.weights_to_bf16(w.float())
        dy = bf(N, T, h, h, c)
        mask = bf(N, T, h, h, c)
        dx = torch.empty_like(dy)
        us = time_us(lambda: conv.conv_dgrad(dy, wd, dy.shape, k=3, mask=mask, out=dx))
        report(f"dgrad conv2 3x3 {c} @{h}", us, 2 * m * 9 * c * c, 2 * (3 * m * c + 9 * c * c))
        del x, y, dy, mask, dx
    # conv3 + residual (1x1, short K) and its dgrad at res4 / res5
    for h, w_, cout in ((28, 128, 512), (14, 256, 1024), (7, 512, 2048)):
        x = bf(N, T, h, h, w_)
        w = bf(cout, 1, 1, w_, scale=w_ ** -0.5)
        b = torch.zeros(cout, device=dev)
        r = bf(N, T, h, h, cout)
        y = torch.empty(N, T, h, h, cout, device=dev, dtype=torch.bfloat16)
        us = time_us(lambda: conv.conv_fwd(x, w, b, relu=True, residual=r, out=y))
        m = N * T * h * h
        report(f"fwd conv3 {w_}->{cout} +res @{h}", us, 2 * m * w_ * cout,
               2 * (m * w_ + 2 * m * cout + w_ * cout))
        wf, wd = conv.weights_to_bf16(w.float())
        dy = bf(N, T, h, h, cout)
        dx = torch.empty(N, T, h, h, w_, device=dev, dtype=torch.bfloat16)
        us = time_us(lambda: conv.conv_dgrad(dy, wd, (N, T, h, h, w_), out=dx))
        report(f"dgrad conv3 {cout}->{w_} @{h}", us, 2 * m * w_ * cout,
               2 * (m * w_ + m * cout + w_ * cout))
        del x, y, r, dy, dx
    # strided projection (im2col 1x1 / s2) at res4 / res5 entry
    for h, cin, cout in ((28, 512, 1024), (14, 1024, 2048)):
        x = bf(N, T, h, h, cin)
        w = bf(cout, 1, 1, cin, scale=cin ** -0.5)
        b = torch.zeros(cout, device=dev)
        ho = h // 2
        y = torch.empty(N, T, ho, ho, cout, device=dev, dtype=torch.bfloat16)
        us = time_us(lambda: conv.conv_fwd(x, w, b, stride=2, out=y))
        m = N * T * ho * ho
        report(f"fwd proj {cin}->{cout} s2 @{h}", us, 2 * m * cin * cout,
               2 * (m * cin + m * cout + cin * cout))
        del x, y
    # weight gradients (+ fused bias gradient) at res3-res5
    for h, cin, cout, k, f in ((56, 256, 64, 1, 32), (56, 64, 256, 1, 0), (56, 64, 64, 1, 8),
                               (56, 256, 128, 1, 32), (28, 512, 128, 1, 64), (28, 128, 512, 1, 0),
                               (28, 128, 128, 3, 0), (14, 256, 256, 3, 0), (7, 512, 512, 3, 0),
                               (14, 1024, 256, 1, 128), (7, 2048, 512, 1, 256),
                               (14, 256, 1024, 1, 0), (7, 512, 2048, 1, 0)):
        x = bf(N, T, h, h, cin)
        dy = bf(N, T, h, h, cout)
        us = time_us(lambda: conv.conv_wgrad(x, dy, k=k, fold=(f, f), bias_grad=True))
        m = N * T * h * h
        report(f"wgrad {k}x{k} {cin}->{cout} @{h}" + (" (shifted x)" if f else ""), us,
               2 * m * k * k * cin * cout, 2 * m * (cin + cout))
        us = time_us(lambda: conv.conv_wgrad(x, dy, k=k, fold=(f, f), bias_grad=False))
        report(f"wgrad {k}x{k} {cin}->{cout} @{h} no-db" + (" (shifted x)" if f else ""), us,
               2 * m * k * k * cin * cout, 2 * m * (cin + cout))
        del x, dy
    if a.json:
        Path(a.json).write_text(json.dumps({"peaks": {"hbm_gbs": hbm, "bf16_tflops": tf},
                                            "rows": rows}, indent=1))


if __name__ == "__main__":
    main()
