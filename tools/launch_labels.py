#!/usr/bin/env python3
"""Per-layer attribution of a train step's kernel launches from the library's
own launch trace (tsm_trace_enable / tsm_trace_dump: the label of the layer
and op that issued each launch, in issue order), joined 1:1 with an ncu
launch list of the same step.

    # on the GPU box: one warm-up step, then one traced step; serialised
    # (TSM_SIDE_STREAM=0) so the launch order is the issue order
    TSM_SIDE_STREAM=0 python tools/launch_labels.py run --out trace.txt
    TSM_SIDE_STREAM=0 ncu --metrics gpu__time_duration.sum --clock-control none \\
        --kernel-name-base demangled -k regex:tsm:: -s <warm-up launches> -c <step launches> \\
        --csv --log-file launches.csv python tools/launch_labels.py run --out trace.txt
    # here
    python tools/launch_labels.py join trace.txt launches.csv [--batch 64]

`run` prints the launch counts ncu needs (it counts with the library's own
launch counter).  `join` prints every labelled launch, the per-op totals and
the forward / backward / other split."""
from __future__ import annotations

import argparse
import collections
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(Path(__file__).resolve().parent))


def run(a):
    import ctypes as C

    import torch

    from paper_1910_00932_b200 import _lib
    from paper_1910_00932_b200.network import TSMNet
    lib = _lib.lib
    lib.tsm_trace_enable.argtypes = [C.c_int]
    lib.tsm_trace_dump.argtypes = [C.c_char_p]
    net = TSMNet(batch=a.batch).init_random(seed=0)
    x = torch.randn(a.batch, 8, 3, 224, 224, device="cuda")
    torch.cuda.synchronize()
    l0 = _lib.launch_count()
    net.train_step(x, lr=1e-13)           # warm-up step
    torch.cuda.synchronize()
    l1 = _lib.launch_count()
    _lib.check(lib.tsm_trace_enable(1))
    net.train_step(x, lr=1e-13)           # traced step
    torch.cuda.synchronize()
    l2 = _lib.launch_count()
    _lib.check(lib.tsm_trace_dump(a.out.encode()))
    _lib.check(lib.tsm_trace_enable(0))
    print(f"launches before the warm-up step: {l0}; warm-up step: {l1 - l0}; traced step: "
          f"{l2 - l1} (ncu: -s {l1} -c {l2 - l1} with -k regex:tsm::)")


def join(a):
    from launch_summary import load
    labels = [l.rstrip("\n") for l in open(a.trace)]
    seq = load(a.launches)
    if len(seq) != len(labels):
        sys.exit(f"launch list has {len(seq)} launches, the trace {len(labels)}: capture the "
                 "traced step exactly (see `run`)")
    tot = sum(v for _, v in seq)
    print(f"# {len(seq)} launches, {tot / 1e3:.1f} µs serialised (cold cache)")
    per_op = collections.OrderedDict()
    for (kern, ns), lab in zip(seq, labels):
        if a.verbose:
            print(f"{ns / 1e3:9.1f} µs  {lab:48s} {kern}")
        key = lab
        per_op.setdefault(key, [0, 0.0, set()])
        per_op[key][0] += 1
        per_op[key][1] += ns
        per_op[key][2].add(kern)
    print("\n# per labelled op (issue order)")
    for lab, (n, ns, kerns) in per_op.items():
        print(f"{ns / 1e3:9.1f} µs n={n:3d}  {lab:48s} {', '.join(sorted(kerns))[:90]}")
    # op classes across units
    cls = collections.defaultdict(float)
    for lab, (n, ns, _) in per_op.items():
        parts = lab.split(" ", 1)
        cls[parts[1] if len(parts) > 1 and parts[0].startswith("res") else lab] += ns
    print("\n# per op class (summed over units)")
    for k, ns in sorted(cls.items(), key=lambda kv: -kv[1]):
        print(f"{ns / 1e3:9.1f} µs {100 * ns / tot:5.1f}%  {k}")
    fwd = sum(ns for lab, (n, ns, _) in per_op.items() if " fwd" in lab or lab.startswith("fwd"))
    bwd = sum(ns for lab, (n, ns, _) in per_op.items() if " bwd" in lab or lab.startswith("bwd")
              or lab.startswith("loss"))
    print(f"\nforward {fwd / 1e3:.1f} µs, backward {bwd / 1e3:.1f} µs, other "
          f"{(tot - fwd - bwd) / 1e3:.1f} µs")


def main():
    ap = argparse.ArgumentParser()
    sub = ap.add_subparsers(dest="cmd", required=True)
    r = sub.add_parser("run")
    r.add_argument("--batch", type=int, default=64)
    r.add_argument("--out", default="trace.txt")
    j = sub.add_parser("join")
    j.add_argument("trace")
    j.add_argument("launches")
    j.add_argument("-v", "--verbose", action="store_true")
    a = ap.parse_args()
    run(a) if a.cmd == "run" else join(a)


if __name__ == "__main__":
    main()
