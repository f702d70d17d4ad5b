#!/usr/bin/env python3
"""Summarise an ncu --csv launch list (gpu__time_duration.sum) by kernel."""
import collections
import csv
import io
import sys


def load(path):
    lines = open(path).read().splitlines()
    start = [i for i, l in enumerate(lines) if l.startswith('"ID"')][0]
    rows = list(csv.DictReader(io.StringIO("\n".join(lines[start:]))))
    seq = []
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", "")) * {"ns": 1, "us": 1e3, "ms": 1e6,
                                                          "nsecond": 1, "usecond": 1e3,
                                                          "msecond": 1e6}[r["Metric Unit"]]
        name = r["Kernel Name"]
        short = name.split("(")[0]
        if "tc_gemm_kernel" in name:
            short = name[name.index("tc_gemm_kernel"):name.index(">") + 1]
        seq.append((short, v))
    return seq


if __name__ == "__main__":
    seq = load(sys.argv[1])
    by = collections.defaultdict(lambda: [0, 0.0])
    for k, v in seq:
        by[k][0] += 1
        by[k][1] += v
    tot = sum(v for _, v in seq)
    print(f"# {len(seq)} launches, total {tot / 1e6:.2f} ms (serialised, cold cache: compare shares)")
    for k, (n, t) in sorted(by.items(), key=lambda kv: -kv[1][1]):
        print(f"{t / 1e6:8.3f} ms {100 * t / tot:5.1f}% n={n:4d} {k}")
    if len(sys.argv) > 2:
        for i, (k, v) in enumerate(seq):
            if v > float(sys.argv[2]) * 1e3:
                print(i, f"{v / 1e3:9.1f} us", k)
