#!/usr/bin/env python3
"""Benchmark for the B200-native TSM hot path.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload shift]
    torchrun --nproc-per-node N bench.py --gpus N ...        (N > 1)
    python bench.py --impl reference ...                     (reference CPU arm)

Prints ONE JSON line on rank 0.

Workload "shift" (BASELINE.json metric part 1, configs[4]): one step = the
temporal shift forward AND its adjoint (kernels.cpp:97-157) over one batch of
synthetic clips per GPU, fold_div = 8, inputs resident in HBM.  Per GPU the
batch is (8, 8, 256, 56, 56) fp32 (the C2 block's input at N=8, 205 MB per
tensor, larger than the 126 MB L2; L2 is also flushed between steps).
Algorithmic bytes per call: elt*N*H*W*(2*C*T - F - B).  Multi-GPU:
each rank shifts its own clips (the shift never crosses clips), no collective
on the data path -> weak scaling.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

SHIFT_SHAPE = (8, 8, 256, 56, 56)
SWEEP_C = (64, 128, 256, 512, 1024, 2048)
SWEEP_T = (8, 16)


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=20)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", choices=["b200", "reference"], default="b200")
    p.add_argument("--workload", choices=["shift"], default="shift")
    p.add_argument("--no-sweep", action="store_true")
    p.add_argument("--no-cpu-baseline", action="store_true")
    return p.parse_args()


# ---------------------------------------------------------------------------
# plumbing

def dist_env():
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    return rank, world, local


def measured_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return {"hbm_gbs": d["hbm_gbs"], "bf16_tflops": d["bf16_tflops"],
                "bf16_tflops_sustained": d.get("bf16_tflops_sustained"), "source": "measured"}
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0,
            "source": "fallback"}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap,utilization.gpu")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [s.strip() for s in line.split(",")]
            if len(parts) >= 8:
                self.rows.append(parts)

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        def num(s):
            try:
                return float(s)
            except ValueError:
                return None
        sm = [num(r[0]) for r in self.rows if num(r[0]) is not None]
        util = [num(r[7]) or 0 for r in self.rows]
        loaded = [s for s, u in zip(sm, util) if u > 50] or sm
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[3 + i] == "Active"})
        return {"sm_mhz": statistics.median(loaded) if loaded else None,
                "sm_max_mhz": num(self.rows[0][1]), "reasons": reasons,
                "samples": len(self.rows)}


def shift_bytes(shape, elt):
    n, t, c, h, w = shape
    f = b = c // 8
    return elt * n * h * w * (2 * c * t - f - b)


# ---------------------------------------------------------------------------
# reference CPU arm (oracle/_ref = the unmodified reference built in place)

def cpu_reference_shift(shape, budget_s=15.0, max_iters=None):
    """Time vidperf::temporal_shift + temporal_shift_adjoint (fp64, OpenMP over
    all host threads) on a bounded sample of `shape`; bytes are counted at the
    workload's fp32 size so the metric matches the GPU arm's."""
    from oracle.oracle import Reference, REF_SO
    ref = Reference()
    n = shape[0]
    sample = (1,) + tuple(shape[1:])
    probe = ref.time_shift(sample, 1, 8, False, False, 1) + ref.time_shift(sample, 1, 8, True,
                                                                            False, 1)
    clips = max(1, min(n, int(budget_s / 4 / max(probe, 1e-6))))
    sample = (clips,) + tuple(shape[1:])
    iters = max(1, min(max_iters or 10**9, int(budget_s / 2 / max(probe * clips, 1e-6))))
    fwd = ref.time_shift(sample, 1, 8, False, False, iters)
    bwd = ref.time_shift(sample, 1, 8, True, False, iters)
    step = fwd + bwd
    gbs = 2 * shift_bytes(sample, 4) / step / 1e9
    cores = int(os.environ.get("OMP_NUM_THREADS", os.cpu_count() or 1))
    return {"value": gbs, "unit": "GB/s", "cores": cores, "kind": "reference",
            "sample": f"vidperf::temporal_shift + temporal_shift_adjoint (fp64, OpenMP "
                      f"{cores} threads) on {sample}, {iters} iters each; fwd {fwd*1e3:.2f} ms, "
                      f"adj {bwd*1e3:.2f} ms; bytes counted at fp32 like the GPU arm",
            "seconds_per_step": step, "lib": str(REF_SO.relative_to(ROOT))}


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    shape = SHIFT_SHAPE
    vals = []
    for _ in range(args.warmup):
        cpu_reference_shift(shape, budget_s=2.0, max_iters=1)
    base = None
    for _ in range(args.steps):
        base = cpu_reference_shift(shape, budget_s=4.0, max_iters=2)
        vals.append(base["seconds_per_step"])
    med = statistics.median(vals)
    value = base["value"] * base["seconds_per_step"] / med
    line = {"impl": "reference", "metric": "shift GB/s", "value": value, "unit": "GB/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": med * 1e3, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": "temporal_shift fwd+adjoint, fold_div=8",
                       "shape_per_gpu": list(shape), "sample": base["sample"]},
            "cpu_baseline": {k: base[k] for k in ("unit", "cores", "kind", "sample")} | {"value": value},
            "e2e": {"value": value, "unit": "GB/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# B200 arm

def run_shift(args):
    import torch
    import torch.distributed as dist

    import paper_1910_00932_b200 as tsm

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    peaks = measured_peaks()
    cfg = tsm.ShiftConfig.fold_div(8)
    stream = torch.cuda.current_stream(dev)

    shape = SHIFT_SHAPE
    g = torch.Generator(device=dev)
    g.manual_seed(1234 + rank)
    x = torch.randn(shape, device=dev, dtype=torch.float32, generator=g)
    y = torch.empty_like(x)
    dx = torch.empty_like(x)
    flush = torch.empty(256 * 1024 * 1024 // 4, device=dev, dtype=torch.float32)
    step_bytes = 2 * shift_bytes(shape, 4)

    def step():
        tsm.temporal_shift(x, cfg, out=y)
        tsm.temporal_shift_adjoint(y, cfg, out=dx)

    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize()

    # Timed region: K steps, each bracketed by events on the launching stream,
    # L2 flushed between steps (outside the events).
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    mids = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    launches0 = tsm.launch_count()
    with ClockSampler(local) as clk:
        for i in range(args.steps):
            flush.fill_(float(i))
            starts[i].record(stream)
            tsm.temporal_shift(x, cfg, out=y)
            mids[i].record(stream)
            tsm.temporal_shift_adjoint(y, cfg, out=dx)
            ends[i].record(stream)
        torch.cuda.synchronize()
    launches = tsm.launch_count() - launches0
    step_ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    fwd_ms = [s.elapsed_time(m) for s, m in zip(starts, mids)]
    total_ms = sum(step_ms)
    t = torch.tensor([total_ms], device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.barrier()
    total_ms = float(t.item())
    ms_per_step = total_ms / args.steps
    value = step_bytes * world / (ms_per_step / 1e3) / 1e9  # whole job GB/s

    # Roofline of the dominant (only) kernel: algorithmic bytes per launch /
    # mean launch duration (forward launches, CUDA events on their stream).
    per_launch = shift_bytes(shape, 4)
    fwd_mean_s = statistics.mean(fwd_ms) / 1e3
    achieved = per_launch / fwd_mean_s / 1e9
    traffic = None
    prof = ROOT / "profiles" / "shift_ncu_traffic.json"
    if prof.exists():
        traffic = json.loads(prof.read_text()).get("dram_bytes_per_launch")
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                "frac": achieved / peaks["hbm_gbs"], "traffic": traffic,
                "kernel": "shift_copy_kernel<int4,4>", "algorithmic_bytes_per_launch": per_launch,
                "peak_source": f"{peaks['source']} hbm_gbs (MEASURED_PEAKS.json, burst)"}

    # e2e through the C ABI with host buffers: H2D + shift + adjoint... the
    # host entry point does H2D, kernel, D2H per call; one step = fwd + adj.
    xh = x.cpu().pin_memory()
    yh = torch.empty_like(xh).pin_memory()
    dxh = torch.empty_like(xh).pin_memory()
    for _ in range(2):
        tsm.temporal_shift_host(xh, cfg, out=yh)
    e2e_steps = max(3, min(args.steps, 10))
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        tsm.temporal_shift_host(xh, cfg, out=yh)
        tsm.temporal_shift_host(yh, cfg, adjoint=True, out=dxh)
    e2e_s = (time.perf_counter() - t0) / e2e_steps
    te = torch.tensor([e2e_s], device=dev)
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_s = float(te.item())
    nbytes = x.numel() * 4
    e2e = {"value": step_bytes * world / e2e_s / 1e9, "unit": "GB/s",
           "h2d_bytes_per_step": 2 * nbytes, "d2h_bytes_per_step": 2 * nbytes,
           "path": "tsm_shift_host (C ABI, pinned host buffers, H2D+kernel+D2H per call)"}

    sweep = None
    if not args.no_sweep and rank == 0:
        sweep = shift_sweep(tsm, torch, dev, stream, peaks)

    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        try:
            c = cpu_reference_shift(shape, budget_s=12.0)
            cpu = {k: c[k] for k in ("value", "unit", "cores", "kind", "sample")}
        except Exception as e:  # reference not built: report, don't fail the bench
            cpu = {"value": None, "unit": "GB/s", "cores": 0, "kind": "reference",
                   "sample": f"unavailable: {e}"}

    if rank == 0:
        line = {
            "metric": "shift GB/s", "value": value, "unit": "GB/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic",
            "config": {"workload": "temporal_shift fwd+adjoint, fold_div=8 (BASELINE configs[4])",
                       "shape_per_gpu": list(shape), "global_clips": shape[0] * world,
                       "l2": "flushed between steps (256 MB write) and inputs > L2",
                       "parallelism": f"dp{world} (clips sharded, no collective)"},
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": launches, "clocks": clk.summary(),
            "fwd_ms_mean": statistics.mean(fwd_ms), "sweep": sweep,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def shift_sweep(tsm, torch, dev, stream, peaks):
    """BASELINE configs[4]: C 64-2048 x T 8/16 x fp32/bf16 at N=8, 56x56."""
    out = []
    cfg = tsm.ShiftConfig.fold_div(8)
    for dtype, elt in ((torch.float32, 4), (torch.bfloat16, 2)):
        for t in SWEEP_T:
            for c in SWEEP_C:
                shape = (8, t, c, 56, 56)
                x = torch.empty(shape, device=dev, dtype=dtype).normal_()
                y = torch.empty_like(x)
                for _ in range(3):
                    tsm.temporal_shift(x, cfg, out=y)
                ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
                reps = 5
                ev[0].record(stream)
                for _ in range(reps):
                    tsm.temporal_shift(x, cfg, out=y)
                ev[1].record(stream)
                torch.cuda.synchronize()
                s = ev[0].elapsed_time(ev[1]) / reps / 1e3
                gbs = shift_bytes(shape, elt) / s / 1e9
                out.append({"C": c, "T": t, "dtype": str(dtype).split(".")[-1],
                            "GBps": round(gbs, 1), "frac": round(gbs / peaks["hbm_gbs"], 3),
                            "us": round(s * 1e6, 1)})
                del x, y
    torch.cuda.empty_cache()
    return out


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
        return
    run_shift(args)


if __name__ == "__main__":
    main()
