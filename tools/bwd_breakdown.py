#!/usr/bin/env python3
"""Backward GEMMs of one train step (capture with TSM_SIDE_STREAM=0 so the
launch order is the issue order) (launch list of exactly one step's worth
of launches, rotated to start at stem_weights), labelled by layer.
Usage: bwd_breakdown.py launches.csv [N]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent))
from launch_summary import load  # noqa: E402

seq = load(sys.argv[1])
N = int(sys.argv[2]) if len(sys.argv) > 2 else 64
s0 = [i for i, (k, _) in enumerate(seq) if "stem_weights" in k][0]
seq = seq[s0:] + seq[:s0]  # no-op for a one-step capture (starts at stem_weights)
b0 = [i for i, (k, _) in enumerate(seq) if "gap_bwd" in k][0]
bwd = seq[b0:]
# layers in backward order (reverse units)
units = []
hin = 56
for (ho, cin0, cout, stride, nb) in [(56, 64, 256, 1, 3), (28, 256, 512, 2, 4),
                                      (14, 512, 1024, 2, 6), (7, 1024, 2048, 2, 3)]:
    for b in range(nb):
        units.append((f"res{len(units) and 0}", ho, cin0 if b == 0 else cout, cout,
                      stride if b == 0 else 1, b == 0, hin if b == 0 else ho))
    hin = ho
T = 8
names = []
for (_, ho, cin, cout, s, first, hi) in reversed(units):
    w = cout // 4
    mo, mi = N * T * ho * ho, N * T * hi * hi
    names += [(f"wgrad c3 {w}->{cout} @{ho}", 2 * mo * w * cout)]
    if first:  # block.cu issues the projection's wgrad right after conv3's
        names += [(f"wgrad proj {cin}->{cout} s{s}", 2 * mo * cin * cout)]
    names += [(f"dgrad c3 @{ho}", 2 * mo * w * cout),
              (f"wgrad c2 3x3 {w} s{s} @{ho}", 2 * mo * 9 * w * w),
              *([(f"dgrad c2 3x3 s1 @{hi}", 2 * mi * 9 * w * w)] if s == 1 else
                [(f"dgrad c2 3x3 s2 @{hi} class {c}", 2 * mo * n * w * w)
                 for c, n in enumerate((1, 2, 2, 4))]),
              (f"wgrad c1 {cin}->{w} @{hi}", 2 * mi * cin * w)]
    if first and s == 1:
        names += [(f"dgrad proj s{s}", 2 * mo * cin * cout),
                  (f"dgrad c1 (+adj shift, +skip) @{hi}", 2 * mi * cin * w)]
    elif first:  # strided projection: its gradient is added onto conv1's in place
        names += [(f"dgrad c1 (+adj shift) @{hi}", 2 * mi * cin * w),
                  (f"dgrad proj s{s} (+= into dx)", 2 * mo * cin * cout)]
    else:
        names += [(f"dgrad c1 (+adj shift, +skip) @{hi}", 2 * mi * cin * w)]
g = [(k, v) for k, v in bwd if "tc_gemm" in k or "halo::" in k]
tot = 0
for (name, fl), (k, v) in zip(names, g):
    us = v / 1e3
    tot += us
    print(f"{name:32s} {k[15:]:18s} {us:8.1f} us {fl / us / 1e6:7.1f} TF/s")
other = sum(v for k, v in bwd if "tc_gemm" not in k and "halo::" not in k) / 1e3
print(f"backward GEMMs {tot:.0f} us; non-GEMM backward kernels {other:.0f} us")
