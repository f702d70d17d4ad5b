#!/usr/bin/env python3
"""Label the backward GEMM launches of a train-step launch list (reverse unit
order) and report per-launch time.  Usage: bwd_breakdown.py launches.csv"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent))
from launch_summary import load  # noqa: E402

seq = load(sys.argv[1])
# backward = from gap_bwd to maxpool_bwd (inclusive), possibly split across the capture window
idx = [i for i, (k, _) in enumerate(seq) if "gap_bwd" in k]
start = idx[0] if idx else 0
end = [i for i, (k, _) in enumerate(seq) if "maxpool_bwd" in k and i > start]
end = end[0] if end else len(seq)
tot = 0.0
cats = {}
for k, v in seq[start:end + 1]:
    tot += v
    key = k if "tc_gemm" not in k else k
    cats[key] = cats.get(key, 0) + v
print(f"backward window: {tot / 1e6:.2f} ms")
for k, v in sorted(cats.items(), key=lambda kv: -kv[1]):
    print(f"{v / 1e6:8.3f} ms  {k}")
