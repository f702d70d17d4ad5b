#!/usr/bin/env python3
"""Per-conv roofline of the forward GEMMs in a train-step launch list
(tools/profile_target.py step at batch N).  Usage: fwd_breakdown.py launches.csv [N]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent))
from launch_summary import load  # noqa: E402


def convs(N=64, T=8):
    out = [("stem (im2col GEMM)", N * T * 112 * 112, 192, 64, 0)]
    hin = 56
    for (ho, cin0, cout, stride, nb) in [(56, 64, 256, 1, 3), (28, 256, 512, 2, 4),
                                          (14, 512, 1024, 2, 6), (7, 1024, 2048, 2, 3)]:
        for b in range(nb):
            cin = cin0 if b == 0 else cout
            w = cout // 4
            hi = hin if b == 0 else ho
            mi, mo = N * T * hi * hi, N * T * ho * ho
            out.append((f"c1 {cin}->{w} @{hi}", mi, cin, w, 0))
            out.append((f"c2 3x3 {w} s{stride if b == 0 else 1}", mo, 9 * w, w, 0))
            if b == 0:
                out.append((f"proj {cin}->{cout} s{stride}", mo, cin, cout, 0))
            out.append((f"c3 {w}->{cout} +res", mo, w, cout, mo * cout))
        hin = ho
    return out


if __name__ == "__main__":
    seq = load(sys.argv[1])
    N = int(sys.argv[2]) if len(sys.argv) > 2 else 64
    i0 = [i for i, (k, v) in enumerate(seq) if "stem_im2col" in k or "stem_s2d" in k][0]
    fw = [(k, v) for k, v in seq[i0:] if "tc_gemm" in k or "halo::" in k]
    tot = ideal = 0
    for (name, M, K, Nn, extra), (k, v) in zip(convs(N), fw):
        us = v / 1e3
        fl = 2 * M * K * Nn
        by = 2 * (M * Nn + K * Nn) + 2 * extra + 2 * M * (K if "3x3" not in name else K // 9)
        best = max(fl / 1.4e15, by / 6.5e12) * 1e6
        tot += us
        ideal += best
        print(f"{name:24s} {us:8.1f} us {fl / us / 1e6:7.1f} TF/s {by / us / 1e3:7.1f} GB/s "
              f" floor {best:6.1f} us  x{us / best:4.1f}")
    print(f"forward GEMMs {tot:.0f} us, roofline floor {ideal:.0f} us")
