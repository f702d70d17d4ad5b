#!/usr/bin/env python3
"""Kernel-level timing of the tcgen05 conv engine and the bottleneck unit
(CUDA events on the launching stream, warm-up first, L2-sized inputs).

    python tools/bench_kernels.py [--json out.json]

Reports per case: ms, TFLOP/s (algorithmic 2*M*N*K), GB/s (algorithmic
bytes: A + B + output, bf16) and the fraction of the attainable roofline
min(P_bf16, I * BW_HBM) with peaks from MEASURED_PEAKS.json."""
from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from paper_1910_00932_b200 import conv  # noqa: E402
from paper_1910_00932_b200.block import Bottleneck  # noqa: E402


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    d = json.loads(p.read_text()) if p.exists() else {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}
    return d["hbm_gbs"], d["bf16_tflops"]


def time_fn(fn, reps=20, warm=5):
    s = torch.cuda.current_stream()
    for _ in range(warm):
        fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(reps):
        fn()
    e1.record(s)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def roof(flops, bytes_, ms, hbm, tf):
    t = ms / 1e3
    attain = min(tf * 1e12, flops / bytes_ * hbm * 1e9)
    return {"ms": round(ms, 4), "TFLOPs": round(flops / t / 1e12, 1),
            "GBps": round(bytes_ / t / 1e9, 1), "intensity": round(flops / bytes_, 1),
            "frac_attainable": round(flops / t / attain, 3),
            "frac_tensor_peak": round(flops / t / (tf * 1e12), 3)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--json")
    a = ap.parse_args()
    hbm, tf = peaks()
    dev = torch.device("cuda")
    out = {"peaks": {"hbm_gbs": hbm, "bf16_tflops": tf}, "conv1_fused": [], "block": []}
    # fused shift + conv1 (1x1): (N, T, H, W, C_in, C_out, F)
    for n, t, h, w, cin, cout, f in [(8, 8, 56, 56, 256, 64, 32), (64, 8, 56, 56, 256, 64, 32),
                                     (8, 8, 14, 14, 1024, 256, 128), (64, 8, 14, 14, 1024, 256, 128),
                                     (64, 8, 7, 7, 2048, 512, 256), (64, 8, 28, 28, 512, 128, 64)]:
        x = torch.randn(n, t, h, w, cin, device=dev).bfloat16()
        wt = (torch.randn(cout, cin, device=dev) / cin ** 0.5).bfloat16()
        b = torch.zeros(cout, device=dev)
        y = torch.empty(n, t, h, w, cout, device=dev, dtype=torch.bfloat16)
        ms = time_fn(lambda: conv.conv1x1_fwd(x, wt, b, fold=(f, f), relu=True, out=y))
        m = n * t * h * w
        r = roof(2 * m * cin * cout, 2 * (m * cin + m * cout + cin * cout), ms, hbm, tf)
        r.update({"shape": [n, t, h, w, cin, cout], "F": f})
        out["conv1_fused"].append(r)
        print("conv1", r, flush=True)
        del x, y
    # bottleneck unit fwd + bwd (C2: C=256, T=8, 56x56)
    for n in (8, 64):
        blk = Bottleneck(256, 256, 1)
        g = torch.Generator(device=dev).manual_seed(0)
        for k, s in blk.shapes().items():
            blk.params[k] = torch.randn(s, device=dev, generator=g) * (0.05 if k[0] == "w" else 0.1)
        x = torch.randn(n, 8, 56, 56, 256, device=dev).bfloat16()
        y = blk.forward(x)
        gy = torch.randn_like(y)
        fwd = time_fn(lambda: blk.forward(x), reps=10, warm=3)
        fb = time_fn(lambda: blk.backward(x, blk.forward(x), gy), reps=10, warm=3)
        flops = 3 * 2 * 1746927616 * n
        r = {"N": n, "fwd_ms": round(fwd, 3), "fwd_bwd_ms": round(fb, 3),
             "clips_per_s": round(n / (fb / 1e3), 1),
             "TFLOPs_fwd_bwd": round(flops / (fb / 1e3) / 1e12, 1)}
        out["block"].append(r)
        print("block", r, flush=True)
        del x, y, gy
    if a.json:
        Path(a.json).write_text(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
