#!/usr/bin/env python3
"""Roofline of every labelled op of the TSM-R50 train step: the launch-label
trace joined with the ncu launch list of the same step (tools/launch_labels.py)
against each op's algorithmic bytes and FLOPs, computed from the network
geometry (build_tsm8f, arch.cpp:140-161; 224 x 224, T = 8, `--batch` clips).

    python tools/step_roofline.py trace.txt launches.csv [--batch 64]

Per op: measured µs (cold-cache, serialised ncu launch list), HBM floor
(algorithmic bytes / measured copy bandwidth), tensor floor (FLOPs / the
sustained bf16 peak — kernels timed inside a long step), the bound that
applies and the fraction of it reached.  Bytes count each tensor once at
bf16 (activations, gradients) plus the 1-bit ReLU masks; FLOPs are the
useful MACs x 2 (no identity-residual or zero-padded-tap work).  The stem
and pool rows count the s2d input through HBM (the stem output, its
gradient and the backward's 4-tap fold stay on chip in the fused kernels)."""
from __future__ import annotations

import argparse
import collections
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(Path(__file__).resolve().parent))

# (stage, units, c_in of unit 0, width, c_out, input extent of unit 0, stride of unit 0)
STAGES = [("res2", 3, 64, 64, 256, 56, 1), ("res3", 4, 256, 128, 512, 56, 2),
          ("res4", 6, 512, 256, 1024, 28, 2), ("res5", 3, 1024, 512, 2048, 14, 2)]


def op_model(batch):
    """label -> (bytes, flops)."""
    T = 8
    px = lambda h: batch * T * h * h  # noqa: E731
    m = {}
    for st, units, c0, w, co, h0, s0 in STAGES:
        for u in range(units):
            ci = c0 if u == 0 else co
            hi = h0 if u == 0 else h0 // s0
            s = s0 if u == 0 else 1
            ho = hi // s
            pi, po = px(hi), px(ho)
            proj = u == 0
            L = f"{st}.{u}"
            bits = lambda p, c: p * c / 8  # noqa: E731
            m[f"{L} fwd shift+c1"] = (2 * pi * (ci + w) + bits(pi, w), 2 * pi * ci * w)
            m[f"{L} fwd c2"] = (2 * (pi + po) * w + bits(po, w), 2 * po * 9 * w * w)
            if proj:
                m[f"{L} fwd proj"] = (2 * po * (ci + co), 2 * po * ci * co)
            m[f"{L} fwd c3+res"] = (2 * po * (w + 2 * co) + bits(po, co), 2 * po * w * co)
            m[f"{L} bwd relu mask"] = (2 * 2 * po * co + bits(po, co), 0)
            m[f"{L} bwd wgrad c3"] = (2 * po * (w + co), 2 * po * w * co)
            m[f"{L} bwd dgrad c3"] = (2 * po * (co + w) + bits(po, w), 2 * po * w * co)
            m[f"{L} bwd wgrad c2"] = (2 * (pi + po) * w, 2 * po * 9 * w * w)
            m[f"{L} bwd dgrad c2"] = (2 * (po + pi) * w + bits(pi, w), 2 * po * 9 * w * w)
            m[f"{L} bwd dgrad c2 (strided, sub-pixel classes)"] = m[f"{L} bwd dgrad c2"]
            m[f"{L} bwd wgrad c1 (shifted x)"] = (2 * pi * (ci + w), 2 * pi * ci * w)
            m[f"{L} bwd dgrad c1 (adjoint shift + skip)"] = (2 * pi * (w + 2 * ci),
                                                              2 * pi * w * ci)
            m[f"{L} bwd dgrad c1 (adjoint shift)"] = (2 * pi * (w + ci), 2 * pi * w * ci)
            if proj:
                m[f"{L} bwd wgrad proj"] = (2 * po * (ci + co), 2 * po * ci * co)
                if s == 1:
                    m[f"{L} bwd dgrad proj"] = (2 * po * (co + ci), 2 * po * ci * co)
                else:  # += into the strided quarter of dx: read + write it
                    m[f"{L} bwd dgrad proj (+= into dx)"] = (2 * po * (co + 2 * ci),
                                                             2 * po * ci * co)
    p1, p2 = px(112), px(56)
    stem_flops = 2 * p1 * 7 * 7 * 3 * 64
    # as implemented: fp32 input -> s2d bf16 (16 ch) -> fused stem conv + pool -> pooled
    # bf16 + argmax bytes (the stem output stays on chip)
    m["fwd stem+pool"] = (batch * T * 3 * 224 * 224 * 4 + 2 * p1 * 16 * 2 + 2 * p2 * 64
                          + p2 * 64, stem_flops)
    # fused pool backward + stem weight gradient: pooled gradient, argmax
    # bytes and the s2d input read once (the stem gradient and the 4-tap fold
    # stay on chip)
    m["bwd pool+stem"] = (2 * p2 * 64 + p2 * 64 + 2 * p1 * 16, stem_flops)
    return m


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("trace")
    ap.add_argument("launches")
    ap.add_argument("--batch", type=int, default=64)
    ap.add_argument("--json")
    a = ap.parse_args()
    from launch_summary import load
    peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
    hbm, tf = peaks["hbm_gbs"], peaks.get("bf16_tflops_sustained", peaks["bf16_tflops"])
    labels = [l.rstrip("\n") for l in open(a.trace)]
    seq = load(a.launches)
    if len(seq) != len(labels):
        sys.exit("launch list and trace differ in length (see tools/launch_labels.py)")
    per = collections.OrderedDict()
    for (_, ns), lab in zip(seq, labels):
        per[lab] = per.get(lab, 0.0) + ns / 1e3
    model = op_model(a.batch)
    tot = sum(per.values())
    rows, cls = [], collections.defaultdict(lambda: [0.0, 0.0])
    print(f"# {tot:.1f} µs serialised; peaks: HBM {hbm} GB/s (copy), bf16 {tf} TF/s "
          f"(sustained)")
    print(f"{'op':52s} {'µs':>8s} {'share':>6s} {'GB':>7s} {'GF':>7s} {'floor':>7s} "
          f"{'bound':>6s} {'frac':>5s}")
    for lab, us in per.items():
        if lab not in model:
            print(f"{lab:52s} {us:8.1f} {100 * us / tot:5.1f}%  (no model)")
            continue
        b, f = model[lab]
        th, tt = b / hbm / 1e3, f / tf / 1e6
        floor = max(th, tt)
        bound = "hbm" if th >= tt else "tensor"
        r = {"op": lab, "us": round(us, 1), "share": round(us / tot, 4), "GB": round(b / 1e9, 3),
             "GFLOP": round(f / 1e9, 2), "floor_us": round(floor, 1), "bound": bound,
             "frac": round(floor / us, 3)}
        rows.append(r)
        print(f"{lab:52s} {us:8.1f} {100 * us / tot:5.1f}% {b / 1e9:7.3f} {f / 1e9:7.1f} "
              f"{floor:7.1f} {bound:>6s} {floor / us:5.2f}")
        k = lab.split(" ", 1)[1] if lab.startswith("res") else lab
        cls[k][0] += us
        cls[k][1] += floor
    print("\n# per op class: measured µs, sum of floors, fraction")
    for k, (us, fl) in sorted(cls.items(), key=lambda kv: -kv[1][0]):
        print(f"{k:46s} {us:8.1f} {fl:8.1f} {fl / us:5.2f}")
    modeled = sum(r["us"] for r in rows)
    floors = sum(r["floor_us"] for r in rows)
    print(f"\nmodeled ops: {modeled:.1f} µs measured, {floors:.1f} µs of floors "
          f"({floors / modeled:.2f}); unmodeled (head, loss, SGD, weights, reductions "
          f"in other labels): {tot - modeled:.1f} µs")
    if a.json:
        Path(a.json).write_text(json.dumps({"total_us": tot, "rows": rows}, indent=1))


if __name__ == "__main__":
    main()
