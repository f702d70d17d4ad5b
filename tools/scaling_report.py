#!/usr/bin/env python3
"""Measured 1 -> N GPU scaling of the DP step next to the reference's own
cluster model (sim.cpp, restated in paper_1910_00932_b200.scaling),
calibrated on this B200 node: utilization from the 1-GPU bench line
(step_tensor.frac), ring bandwidth / latency from tools/nccl_allreduce.py.

    python tools/scaling_report.py [profiles/r01] > profiles/r01/scaling_model.txt
"""
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_1910_00932_b200 import scaling as sc  # noqa: E402

d = Path(sys.argv[1]) if len(sys.argv) > 1 else ROOT / "profiles" / "r01"
lines = {}
for f in sorted(d.glob("bench_train_n*_latest.json.log")):
    j = json.loads(f.read_text().strip().splitlines()[-1])
    lines[j["n_gpus"]] = j
ar = [json.loads(x) for x in (d / "nccl_allreduce.json").read_text().splitlines() if x.strip()]
n1 = lines[1]
util = n1["step_tensor"]["frac"]
# ring bandwidth: the largest measured world; latency: solve the 25 MB and
# full-size points of that world for (latency, bandwidth) of the Ring formula
big = max(ar, key=lambda r: r["world"])
w = big["world"]
f_full, f_b = big["full"], big["bucket25MB"]
k = 2 * (w - 1) / w
bw = k * (f_full["bytes"] - f_b["bytes"]) / (f_full["seconds"] - f_b["seconds"])
lat = max(0.0, (f_full["seconds"] - k * f_full["bytes"] / bw) / (2 * (w - 1)))
print("# DP step scaling: measured vs the reference's cluster model (sim.cpp)")
print(f"# calibration: peak {sc.b200_profile().peak_flops_per_gpu / 1e12:.1f} TF/s (sustained bf16),"
      f" utilization {util:.3f} (1-GPU step), ring bw {bw / 1e9:.0f} GB/s, hop latency {lat * 1e6:.1f} us"
      f" (NCCL allreduce, {w} GPUs)")
# the reference's observed_scalability is baseline / (p * time(p)) for a
# fixed total amount of work; the bench is weak-scaled (64 clips per GPU), so
# the wall time of the 1-GPU step's work at p GPUs is ms_per_step(p) / p
timings = [(n, lines[n]["ms_per_step"] * 1e-3 / n) for n in sorted(lines)]
obs = dict(sc.observed_scalability(timings))
print(f"{'gpus':>4} {'clips/s':>9} {'ms/step':>8} {'observed':>8} | {'model (ref, no overlap)':>24} {'model (bucket overlap)':>23}")
for n in sorted(lines):
    p = sc.b200_profile(nodes=n, utilization=util, net_latency=lat, net_bandwidth=bw)
    a = sc.step_time(p, per_gpu_batch=64)
    b = sc.step_time_overlapped(p, per_gpu_batch=64)
    base = sc.step_time(sc.with_nodes(p, 1), per_gpu_batch=64).t_step
    print(f"{n:>4} {lines[n]['value']:>9.1f} {lines[n]['ms_per_step']:>8.2f} {obs[n]:>8.3f} |"
          f" {a.t_step * 1e3:>8.2f} ms  scal {base / a.t_step:>6.3f}   {b.t_step * 1e3:>8.2f} ms  scal {base / b.t_step:>6.3f}")
