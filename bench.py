#!/usr/bin/env python3
"""Benchmark for the B200-native TSM hot path.  Prints ONE JSON line on rank 0.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload train|shift]
    python -m torch.distributed.run --nproc-per-node N bench.py --gpus N ...
    python bench.py --impl reference ...          (the reference CPU arm)

Workload "train" (default; BASELINE metric "TSM-R50 8f train clips/sec at
1/2/4/8 B200", configs[3]): one step = TSM-ResNet-50 8-frame 224x224
forward + Sigma-y^2 loss + backward + bucketed NCCL gradient allreduce
(overlapped with backward) + momentum-SGD update, 64 synthetic clips per GPU
(weak scaling: the batch is sharded, per-GPU work fixed).  Inputs (308 MB
per step per GPU) are larger than the 126 MB L2.

Workload "shift" (BASELINE metric part 1, configs[4]): temporal shift forward
+ adjoint on (8, 8, 256, 56, 56) fp32 per GPU; no collective.

Workload "block" (BASELINE configs[1]): one residual-shift bottleneck unit
(C=256, T=8, 56x56; kernel_bench.cpp:62-72 shape) forward + backward through
tsm_block_fwd / tsm_block_bwd at --batch clips per GPU (8 and 64 are the
recorded points), against the attainable roofline of its op sequence and the
reference's own block op sequence on the host cores at N=1.
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
if os.environ.get("TSM_PKG_ROOT"):  # A/B of another build of the package on the same box
    sys.path.insert(0, os.environ["TSM_PKG_ROOT"])

TRAIN_BATCH = 64            # clips per GPU, BASELINE configs[3]
TRAIN_FLOP_PER_CLIP = 3 * 2 * 32697909248   # 3 x fwd (sim.hpp:38-39); MACs cost_test.cpp:68
SHIFT_SHAPE = (8, 8, 256, 56, 56)
REF_SAMPLE_HW = 112         # reference CPU arm: one clip at 112x112 (1/4 of the pixels)
SWEEP_C = (64, 128, 256, 512, 1024, 2048)
SWEEP_T = (8, 16)


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=20)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", choices=["b200", "reference"], default="b200")
    p.add_argument("--workload", choices=["train", "shift", "block"], default="train")
    p.add_argument("--batch", type=int, default=None,
                   help="clips per GPU (train: 64, block: 8)")
    p.add_argument("--no-sweep", action="store_true")
    p.add_argument("--graph", choices=["auto", "on", "off"], default="auto",
                   help="train: CUDA-graph replay of the step (auto: on for batch <= 16)")
    p.add_argument("--no-cpu-baseline", action="store_true")
    return p.parse_args()


# ---------------------------------------------------------------------------
# plumbing

def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def measured_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return {"hbm_gbs": d["hbm_gbs"], "bf16_tflops": d["bf16_tflops"],
                "bf16_tflops_sustained": d.get("bf16_tflops_sustained", d["bf16_tflops"]),
                "source": "measured"}
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0,
            "source": "fallback"}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap,utilization.gpu")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, index: int):
        self.index, self.rows, self.proc = index, [], None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
            # nvidia-smi takes ~0.1-0.5 s to start: wait for its first line so
            # the timed region is sampled from its start, then keep only
            # samples taken inside it
            t0 = time.perf_counter()
            while not self.rows and time.perf_counter() - t0 < 3.0 and self.proc.poll() is None:
                time.sleep(0.01)
            self.rows = []
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
        def num(s):
            try:
                return float(s)
            except ValueError:
                return None
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [num(r[0]) for r in self.rows]
        util = [num(r[7]) or 0 for r in self.rows]
        loaded = [s for s, u in zip(sm, util) if s is not None and u > 50] or \
            [s for s in sm if s is not None]
        reasons = sorted({self.NAMES[i] for r in self.rows for i in range(4) if r[3 + i] == "Active"})
        power = [num(r[2]) for r in self.rows if num(r[2]) is not None]
        return {"sm_mhz": statistics.median(loaded) if loaded else None,
                "sm_max_mhz": num(self.rows[0][1]), "reasons": reasons,
                "power_w_max": max(power) if power else None, "samples": len(self.rows)}


def shift_bytes(shape, elt):
    n, t, c, h, w = shape
    f = b = c // 8
    return elt * n * h * w * (2 * c * t - f - b)


def latest_profile(name):
    """profiles/rNN/<name> of the most recent round that has it."""
    cands = sorted((ROOT / "profiles").glob(f"r*/{name}"))
    return cands[-1] if cands else ROOT / "profiles" / name


def allreduce_max(x, dist, world, dev):
    import torch
    t = torch.tensor([float(x)], device=dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# ---------------------------------------------------------------------------
# reference CPU arm: oracle/_ref = the unmodified reference built in place

def cpu_reference_train(hw=REF_SAMPLE_HW, ref=None, iters=1):
    """vidperf::Network::loss_gradients on 1 clip of build_tsm8f() with the
    input extent set to hw x hw, OpenMP over all host threads; clips/s scaled
    to 224x224 by the pixel ratio (conv work is linear in pixels)."""
    from oracle.oracle import Reference
    secs = (ref or Reference()).time_train_clip(hw, hw, clips=1, iters=iters)
    scale = (hw * hw) / (224.0 * 224.0)
    cores = int(os.environ.get("OMP_NUM_THREADS", os.cpu_count() or 1))
    return {"value": scale / secs, "unit": "clips/s", "cores": cores, "kind": "reference",
            "sample": f"vidperf::Network(build_tsm8f).loss_gradients on 1 clip of "
                      f"8x3x{hw}x{hw} (fp64, OpenMP {cores} threads): {secs:.2f} s = "
                      f"{hw * hw}/{224 * 224} of a 224x224 clip's pixels", "seconds": secs}


def train_config(B, world, opt):
    """The `config` object of the train workload, identical in both arms."""
    return {"workload": "TSM-ResNet-50 8-frame 224x224 training step: fwd + sum-of-squares "
                        "loss + bwd + NCCL bucketed gradient allreduce (overlapped) + momentum "
                        "SGD (BASELINE configs[3])",
            "model": "tsm8f (build_tsm8f, shift 1/8)", "global_batch": B * world,
            "batch_per_gpu": B, "seq_len": 8, "parallelism": f"dp{world}",
            "l2": "inputs (308 MB/step/GPU) larger than L2", "optimizer": opt}


TRAIN_OPT = dict(lr=1e-13, momentum=0.9, weight_decay=1e-4)


def shift_config(shape, world):
    return {"workload": "temporal_shift fwd+adjoint, fold_div=8 (configs[4])",
            "shape_per_gpu": list(shape), "parallelism": f"dp{world}",
            "l2": "inputs (205 MB) larger than L2"}


def cpu_reference_shift(shape, budget_s=12.0, max_iters=None):
    """vidperf::temporal_shift + temporal_shift_adjoint (fp64, OpenMP) on a
    bounded sample of `shape`; bytes counted at fp32 like the GPU arm."""
    from oracle.oracle import Reference
    ref = Reference()
    sample = (1,) + tuple(shape[1:])
    probe = ref.time_shift(sample, 1, 8, False, False, 1) + ref.time_shift(sample, 1, 8, True,
                                                                            False, 1)
    clips = max(1, min(shape[0], int(budget_s / 4 / max(probe, 1e-6))))
    sample = (clips,) + tuple(shape[1:])
    iters = max(1, min(max_iters or 10**9, int(budget_s / 2 / max(probe * clips, 1e-6))))
    fwd = ref.time_shift(sample, 1, 8, False, False, iters)
    bwd = ref.time_shift(sample, 1, 8, True, False, iters)
    cores = int(os.environ.get("OMP_NUM_THREADS", os.cpu_count() or 1))
    return {"value": 2 * shift_bytes(sample, 4) / (fwd + bwd) / 1e9, "unit": "GB/s",
            "cores": cores, "kind": "reference", "seconds": fwd + bwd,
            "sample": f"vidperf::temporal_shift + temporal_shift_adjoint (fp64, OpenMP {cores} "
                      f"threads) on {sample}, {iters} iters each; bytes counted at fp32"}


def run_reference(args):
    """The reference arm: the unmodified reference (oracle/_ref, built in place
    from /root/reference) on this box's host cores, rank 0 only.

    train: one timed step = one Network::loss_gradients (fwd + Sigma-y^2 loss
    + bwd, fp64, OpenMP over all host threads) on one clip of build_tsm8f()
    at 112x112 — 1/4 of a 224x224 clip's pixels, so a step is 1/4 of a clip
    of the configured workload and `value` = (1/4) / step time (clips/s).
    `ms_per_step` is the time actually measured per step.  The pixel scaling
    is checked once per run (outside the timed steps) against one full
    224x224 clip: `scaling_check`.  (A 224x224 clip takes minutes on the
    host, so K of them would not fit the run.)"""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    if args.workload == "block":
        return run_reference_block(args)
    from oracle.oracle import Reference
    ref = Reference()
    secs = []
    if args.workload == "train":
        B = args.batch or TRAIN_BATCH
        for _ in range(args.warmup):
            cpu_reference_train(ref=ref)
        for _ in range(args.steps):
            secs.append(cpu_reference_train(ref=ref)["seconds"])
        ms = statistics.mean(secs) * 1e3
        frac = REF_SAMPLE_HW ** 2 / 224.0 ** 2
        value = frac / (ms / 1e3)
        full = ref.time_train_clip(224, 224, clips=1, iters=1)
        cores = int(os.environ.get("OMP_NUM_THREADS", os.cpu_count() or 1))
        sample = (f"vidperf::Network(build_tsm8f).loss_gradients (fp64, OpenMP {cores} threads) "
                  f"on 1 clip of 8x3x{REF_SAMPLE_HW}x{REF_SAMPLE_HW} per step = "
                  f"{REF_SAMPLE_HW ** 2}/{224 ** 2} of a 224x224 clip")
        metric, unit = "TSM-R50 8f train clips/sec", "clips/s"
        cfg = train_config(B, world, TRAIN_OPT)
        extra = {"scaling_check": {
            "full_224_clip_s": full, "extrapolated_224_clip_s": (ms / 1e3) / frac,
            "ratio_measured_over_extrapolated": full / ((ms / 1e3) / frac),
            "clips_per_s_full_224": 1.0 / full}}
    else:
        for _ in range(args.warmup):
            cpu_reference_shift(SHIFT_SHAPE, 2.0, 1)
        base = None
        vals = []
        for _ in range(args.steps):
            base = cpu_reference_shift(SHIFT_SHAPE, 4.0, 2)
            vals.append(base["value"])
            secs.append(base["seconds"])
        value = statistics.median(vals)
        ms = statistics.mean(secs) * 1e3
        cores, sample = base["cores"], base["sample"]
        metric, unit = "shift GB/s", "GB/s"
        cfg = shift_config(SHIFT_SHAPE, world)
        extra = {}
    line = {"impl": "reference", "metric": metric, "value": value, "unit": unit,
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": cfg,
            "cpu_baseline": {"value": value, "unit": unit, "cores": cores,
                             "kind": "reference", "sample": sample},
            "e2e": {"value": value, "unit": unit, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}, **extra}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# B200 arm

def setup_dist():
    import torch
    import torch.distributed as dist
    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    return torch, dist, rank, world, local, dev


def conv1_roofline(torch, dev, peaks, batch):
    """The north-star kernel: fused shift + 1x1 conv of a res2 unit
    (C=256 -> 64, F=32, 56x56, T=8) at the step's batch; HBM-bound.
    Algorithmic bytes per launch = bf16 (x + y + w) = 2*(M*K + M*N + K*N)."""
    from paper_1910_00932_b200 import conv
    n, t, h, w, cin, cout, f = batch, 8, 56, 56, 256, 64, 32
    x = torch.randn(n, t, h, w, cin, device=dev).bfloat16()
    wt = (torch.randn(cout, cin, device=dev) / 16).bfloat16()
    b = torch.zeros(cout, device=dev)
    y = torch.empty(n, t, h, w, cout, device=dev, dtype=torch.bfloat16)
    flush = torch.empty(64 * 1024 * 1024, device=dev)
    s = torch.cuda.current_stream(dev)
    for _ in range(3):
        conv.conv1x1_fwd(x, wt, b, fold=(f, f), relu=True, out=y)
    times = []
    for _ in range(10):
        flush.fill_(1.0)                      # 256 MB write: L2 flushed between launches
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        conv.conv1x1_fwd(x, wt, b, fold=(f, f), relu=True, out=y)
        e1.record(s)
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1) / 1e3)
    m = n * t * h * w
    nbytes = 2 * (m * cin + m * cout + cin * cout)
    flops = 2 * m * cin * cout
    mean = statistics.mean(times)
    achieved = nbytes / mean / 1e9
    traffic = None
    prof = latest_profile("conv1_fused_ncu.json")
    if prof.exists():
        traffic = json.loads(prof.read_text()).get("dram_bytes_per_launch")
    return {"bound": "hbm", "achieved": achieved, "peak": peaks["hbm_gbs"], "unit": "GB/s",
            "frac": achieved / peaks["hbm_gbs"], "traffic": traffic,
            "kernel": "tc_gemm_kernel<BN=64,KCA=32> fused temporal shift + 1x1 conv (res2 conv1)",
            "shape": {"N": n, "T": t, "HW": h * w, "c_in": cin, "c_out": cout, "F": f},
            "algorithmic_bytes_per_launch": nbytes, "launch_us_mean": mean * 1e6,
            "tflops": flops / mean / 1e12,
            "peak_source": f"{peaks['source']} hbm_gbs (MEASURED_PEAKS.json, burst: timed alone)"}


def shift_summary(torch, dev, peaks):
    import paper_1910_00932_b200 as tsm
    cfg = tsm.ShiftConfig.fold_div(8)
    x = torch.randn(SHIFT_SHAPE, device=dev)
    y = torch.empty_like(x)
    s = torch.cuda.current_stream(dev)
    for _ in range(3):
        tsm.temporal_shift(x, cfg, out=y)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(10):
        tsm.temporal_shift(x, cfg, out=y)
        tsm.temporal_shift_adjoint(y, cfg, out=x)
    e1.record(s)
    torch.cuda.synchronize()
    sec = e0.elapsed_time(e1) / 1e3 / 20
    gbs = shift_bytes(SHIFT_SHAPE, 4) / sec / 1e9
    return {"shape": list(SHIFT_SHAPE), "dtype": "f32", "GBps": gbs,
            "frac": gbs / peaks["hbm_gbs"], "us": sec * 1e6}


def in_step_roofline(probe, peaks, alone):
    """The north-star kernel timed inside the timed steps: CUDA events on the
    block's stream around each res2 fused shift + conv1 launch (C ABI probe).
    In the step the kernel also writes conv1's ReLU bitmask (1 bit per
    output), so its algorithmic bytes per launch are bf16 (x + y + w) +
    M*64/8.  `alone` (the same kernel timed by itself, L2 flushed between
    launches) is kept as a sub-object."""
    n, us, m = probe
    if n == 0:
        raise RuntimeError("in-step probe recorded no fused shift + conv1 launch")
    cin, cout = 256, 64
    nbytes = 2 * (m * cin + m * cout + cin * cout) + m * cout // 8
    achieved = nbytes / (us / 1e6) / 1e9
    return {"bound": "hbm", "achieved": achieved, "peak": peaks["hbm_gbs"], "unit": "GB/s",
            "frac": achieved / peaks["hbm_gbs"], "traffic": alone["traffic"],
            "kernel": alone["kernel"] + ", timed inside the training step",
            "shape": alone["shape"], "algorithmic_bytes_per_launch": nbytes,
            "launch_us_mean": us, "launches_timed": n,
            "tflops": 2 * m * cin * cout / (us / 1e6) / 1e12,
            "peak_source": f"{peaks['source']} hbm_gbs (MEASURED_PEAKS.json copy bandwidth; "
                           "no sustained HBM figure is recorded)",
            "timed_alone": {k: alone[k] for k in ("achieved", "frac", "launch_us_mean",
                                                  "algorithmic_bytes_per_launch", "tflops")}}


def run_train(args):
    torch, dist, rank, world, local, dev = setup_dist()
    import paper_1910_00932_b200 as tsm
    from paper_1910_00932_b200.network import TSMNet

    peaks = measured_peaks()
    B = args.batch or TRAIN_BATCH
    net = TSMNet(batch=B, device=dev).init_random(seed=0)   # identical init on every rank
    if world > 1:
        net.dp_init()
    # small batches are launch-bound (~2,550 kernels per step): replay the
    # captured step as one CUDA graph (single GPU; the library runs data-
    # parallel steps eagerly)
    graph = args.graph == "on" or (args.graph == "auto" and B <= 16 and world == 1)
    if graph:
        net.set_graph(True)
    g = torch.Generator(device=dev).manual_seed(1000 + rank)
    x = torch.randn((B, 8, 3, 224, 224), device=dev, generator=g)
    # Sigma-y^2 loss without BN gives O(1e10) gradients: a tiny lr keeps the
    # weights finite while the update still runs every step.
    opt = TRAIN_OPT
    s = torch.cuda.current_stream(dev)

    for _ in range(max(args.warmup, 3)):
        net.train_step(x, **opt)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    from paper_1910_00932_b200 import _lib
    # events around the res2 fused shift + conv1 launches inside the timed
    # steps (eager steps only: a graph replay bypasses the host-side probe)
    if not graph:
        _lib.probe_shift_conv1(256, 64)
    l0 = tsm.launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        e0.record(s)
        for _ in range(args.steps):
            net.train_step(x, **opt)
        e1.record(s)
        torch.cuda.synchronize()
    launches = tsm.launch_count() - l0
    if graph:   # graph mode: the probe runs on 3 eager steps after the timed region
        _lib.probe_shift_conv1(256, 64)
        for _ in range(3):
            net.train_step(x, **opt)
        torch.cuda.synchronize()
    _lib.probe_shift_conv1(0)
    probe = _lib.probe_shift_conv1_read()
    if world > 1:
        dist.barrier()
    ms = allreduce_max(e0.elapsed_time(e1), dist, world, dev) / args.steps
    value = B * world / (ms / 1e3)
    loss_val = float(net.loss.item())

    # e2e through the public API: every step copies its clips from pinned host
    # memory to the device and reads its loss back.  As a training input
    # pipeline would, the copy for step i+1 runs on a copy stream into the
    # second of two device buffers while step i computes (each buffer is
    # reused only after the step that read it has finished).
    xh = x.cpu().pin_memory()
    xd = [torch.empty_like(x), torch.empty_like(x)]
    cs = torch.cuda.Stream(dev)
    ready = [torch.cuda.Event(), torch.cuda.Event()]
    freed = [torch.cuda.Event(), torch.cuda.Event()]

    def prefetch(i):
        b = i % 2
        with torch.cuda.stream(cs):
            cs.wait_event(freed[b])
            xd[b].copy_(xh, non_blocking=True)
            ready[b].record(cs)

    # each step's loss is copied to pinned host memory behind the step and
    # read on the host one step later: the host enqueues step i + 1 before it
    # waits for step i's result, as an input pipeline would
    lh = torch.empty(2, dtype=net.loss.dtype, pin_memory=True)
    done = [torch.cuda.Event(), torch.cuda.Event()]
    losses = []

    def e2e_run(n):
        prefetch(0)
        pending = None
        for i in range(n):
            b = i % 2
            torch.cuda.current_stream(dev).wait_event(ready[b])
            loss = net.train_step(xd[b], **opt)
            freed[b].record()
            lh[b].copy_(loss.reshape(1)[0], non_blocking=True)  # D2H of the step's result
            done[b].record()
            if i + 1 < n:
                prefetch(i + 1)
            if pending is not None:
                done[pending].synchronize()
                losses.append(float(lh[pending]))
            pending = b
        done[pending].synchronize()
        losses.append(float(lh[pending]))

    e2e_steps = max(3, args.steps)  # (the first copy is not overlapped: amortise it)
    e2e_run(2)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    e2e_run(e2e_steps)
    e2e_s = allreduce_max((time.perf_counter() - t0) / e2e_steps, dist, world, dev)
    e2e = {"value": B * world / e2e_s, "unit": "clips/s", "h2d_bytes_per_step": xh.numel() * 4,
           "d2h_bytes_per_step": 4,
           "path": "TSMNet.train_step (C ABI tsm_net_train_step); each step's clips copied from "
                   "pinned host memory (copy of step i+1 overlapped with step i on a copy "
                   "stream, double-buffered) and its loss copied back to pinned host memory "
                   "and read by the host one step later"}

    extra = {}
    if rank == 0:
        extra["roofline"] = in_step_roofline(probe, peaks, conv1_roofline(torch, dev, peaks, B))
        if graph:
            extra["roofline"]["kernel"] += " (eager steps right after the graph-replayed timed steps)"
        extra["shift"] = shift_summary(torch, dev, peaks)
        if not args.no_cpu_baseline and world == 1:
            try:
                c = cpu_reference_train()
                extra["cpu_baseline"] = {k: c[k] for k in ("value", "unit", "cores", "kind",
                                                            "sample")}
            except Exception as exc:  # reference not built: report, don't fail
                extra["cpu_baseline"] = {"value": None, "unit": "clips/s", "cores": 0,
                                         "kind": "reference", "sample": f"unavailable: {exc}"}
    step_tflops = TRAIN_FLOP_PER_CLIP * B / (ms / 1e3) / 1e12
    if rank == 0:
        line = {
            "metric": "TSM-R50 8f train clips/sec", "value": value, "unit": "clips/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic clips N(0,1), random-init weights (init_conv distributions)",
            "config": train_config(B, world, opt), "cuda_graph": graph,
            "roofline": extra.get("roofline"),
            "step_tensor": {"achieved_tflops": step_tflops,
                            "peak_tflops": peaks["bf16_tflops_sustained"],
                            "frac": step_tflops / peaks["bf16_tflops_sustained"],
                            "flop_per_clip": TRAIN_FLOP_PER_CLIP,
                            "peak_source": f"{peaks['source']} bf16_tflops_sustained"},
            "cpu_baseline": extra.get("cpu_baseline"), "e2e": e2e, "gpu_launches": launches,
            "clocks": clk.summary(), "loss": loss_val, "shift": extra.get("shift"),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def run_shift(args):
    torch, dist, rank, world, local, dev = setup_dist()
    import paper_1910_00932_b200 as tsm
    peaks = measured_peaks()
    cfg = tsm.ShiftConfig.fold_div(8)
    s = torch.cuda.current_stream(dev)
    shape = SHIFT_SHAPE
    g = torch.Generator(device=dev).manual_seed(1234 + rank)
    x = torch.randn(shape, device=dev, generator=g)
    y, dx = torch.empty_like(x), torch.empty_like(x)
    step_bytes = 2 * shift_bytes(shape, 4)
    for _ in range(max(args.warmup, 3)):
        tsm.temporal_shift(x, cfg, out=y)
        tsm.temporal_shift_adjoint(y, cfg, out=dx)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    l0 = tsm.launch_count()
    # repeat the K-step timed loop until >= 1 s so the clock sampler sees load
    reps, total_ms, fwd = 0, 0.0, []
    with ClockSampler(local) as clk:
        t_start = time.perf_counter()
        while reps == 0 or time.perf_counter() - t_start < 1.0:
            ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True),
                   torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
            for a, m, b in ev:
                a.record(s)
                tsm.temporal_shift(x, cfg, out=y)
                m.record(s)
                tsm.temporal_shift_adjoint(y, cfg, out=dx)
                b.record(s)
            torch.cuda.synchronize()
            total_ms += sum(a.elapsed_time(b) for a, _, b in ev)
            fwd += [a.elapsed_time(m) for a, m, _ in ev]
            reps += 1
    launches = (tsm.launch_count() - l0) // reps
    ms = allreduce_max(total_ms / (reps * args.steps), dist, world, dev)
    value = step_bytes * world / (ms / 1e3) / 1e9
    per_launch = shift_bytes(shape, 4)
    achieved = per_launch / (statistics.mean(fwd) / 1e3) / 1e9
    traffic = None
    prof = latest_profile("shift_ncu.json")
    if prof.exists():
        traffic = json.loads(prof.read_text()).get("dram_bytes_per_launch")
    xh, yh, dxh = x.cpu().pin_memory(), torch.empty(shape).pin_memory(), torch.empty(shape).pin_memory()
    tsm.temporal_shift_host(xh, cfg, out=yh)
    t0 = time.perf_counter()
    for _ in range(3):
        tsm.temporal_shift_host(xh, cfg, out=yh)
        tsm.temporal_shift_host(yh, cfg, adjoint=True, out=dxh)
    e2e_s = allreduce_max((time.perf_counter() - t0) / 3, dist, world, dev)
    if rank == 0:
        cpu = None
        if not args.no_cpu_baseline and world == 1:
            try:
                c = cpu_reference_shift(shape)
                cpu = {k: c[k] for k in ("value", "unit", "cores", "kind", "sample")}
            except Exception as exc:
                cpu = {"value": None, "unit": "GB/s", "cores": 0, "kind": "reference",
                       "sample": f"unavailable: {exc}"}
        line = {"metric": "shift GB/s", "value": value, "unit": "GB/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
                "data": "synthetic",
                "config": shift_config(shape, world),
                "roofline": {"bound": "hbm", "achieved": achieved, "peak": peaks["hbm_gbs"],
                             "unit": "GB/s", "frac": achieved / peaks["hbm_gbs"],
                             "traffic": traffic, "kernel": "shift_copy_kernel<int4,4>",
                             "algorithmic_bytes_per_launch": per_launch},
                "cpu_baseline": cpu,
                "e2e": {"value": step_bytes * world / e2e_s / 1e9, "unit": "GB/s",
                        "h2d_bytes_per_step": 2 * x.numel() * 4,
                        "d2h_bytes_per_step": 2 * x.numel() * 4},
                "gpu_launches": launches, "clocks": clk.summary(),
                "sweep": None if args.no_sweep else shift_sweep(tsm, torch, dev, s, peaks)}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


# ---------------------------------------------------------------------------
# block workload (BASELINE configs[1])

BLOCK = dict(c=256, t=8, h=56, w=56)


def block_config(B, world):
    return {"workload": "residual-shift TSM bottleneck unit forward + backward (BASELINE "
                        "configs[1]): C=256 -> width 64 -> 256, T=8, 56x56, shift 1/8 "
                        "(F=B=32), identity skip; tsm_block_fwd + tsm_block_bwd",
            "batch_per_gpu": B, "global_batch": B * world, "seq_len": BLOCK["t"],
            "parallelism": f"dp{world} (independent clips, no exchange)",
            "l2": f"activations ({B * 8 * 3136 * 256 * 2 / 1e6:.0f} MB per tensor) "
                  f"{'larger' if B >= 8 else 'smaller'} than L2"}


def block_ops(m):
    """Algorithmic work of the unit's op sequence for m pixels (rows): per
    op (name, FLOPs, HBM bytes) with bf16 tensors, fp32 weights/bias grads.
    Forward: run_unit (net.cpp:85-126); backward: loss_gradients' reverse
    sweep for one unit (net.cpp:184-248), starting from gy (the ReLU
    backward of the residual output reads gy and y)."""
    c, w = BLOCK["c"], BLOCK["c"] // 4
    e = 2
    W1, W2, W3 = c * w, 9 * w * w, w * c
    return [
        # forward
        ("fwd shift+conv1 1x1 256->64 +relu", 2 * m * c * w, e * (m * c + m * w + W1)),
        ("fwd conv2 3x3 64->64 +relu", 2 * m * 9 * w * w, e * (2 * m * w + W2)),
        ("fwd conv3 1x1 64->256 +skip +relu", 2 * m * w * c, e * (m * w + 2 * m * c + W3)),
        # backward
        ("bwd relu mask of y", 0, e * 3 * m * c),
        ("bwd dgrad conv3", 2 * m * c * w, e * (m * c + m * w + W3)),
        ("bwd wgrad conv3 (+db3)", 2 * m * c * w, e * (m * c + m * w) + 4 * W3),
        ("bwd dgrad conv2", 2 * m * 9 * w * w, e * (2 * m * w + W2)),
        ("bwd wgrad conv2 (+db2)", 2 * m * 9 * w * w, e * 2 * m * w + 4 * W2),
        ("bwd dgrad conv1 + adjoint shift + skip grad", 2 * m * w * c,
         e * (m * w + 2 * m * c + W1)),
        ("bwd wgrad conv1 on shifted x (+db1)", 2 * m * w * c, e * (m * c + m * w) + 4 * W1),
    ]


def run_block(args):
    torch, dist, rank, world, local, dev = setup_dist()
    import paper_1910_00932_b200 as tsm
    from paper_1910_00932_b200.block import Bottleneck
    peaks = measured_peaks()
    B = args.batch or 8
    c, t, h, w = BLOCK["c"], BLOCK["t"], BLOCK["h"], BLOCK["w"]
    g = torch.Generator(device=dev).manual_seed(77 + rank)
    blk = Bottleneck(c, c, 1, tsm.ShiftConfig.fold_div(8), device=dev)
    for k, shp in blk.shapes().items():   # init_conv distributions (net.cpp:14-22)
        fan = shp[1] * shp[2] * shp[3] if len(shp) == 4 else 1
        std = (2.0 / fan) ** 0.5 if k.startswith("w") else 0.1
        blk.params[k] = torch.randn(shp, device=dev, generator=g) * std
    x = torch.randn((B, t, h, w, c), device=dev, generator=g).bfloat16()
    gy = torch.randn((B, t, h, w, c), device=dev, generator=g).bfloat16()
    s = torch.cuda.current_stream(dev)
    for _ in range(max(args.warmup, 3)):
        y = blk.forward(x)
        blk.backward(x, y, gy)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    l0 = tsm.launch_count()
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(args.steps)]
    with ClockSampler(local) as clk:
        for a, m_, b in ev:
            a.record(s)
            y = blk.forward(x)
            m_.record(s)
            blk.backward(x, y, gy)
            b.record(s)
        torch.cuda.synchronize()
    launches = tsm.launch_count() - l0
    fwd_ms = statistics.mean(a.elapsed_time(m_) for a, m_, _ in ev)
    bwd_ms = statistics.mean(m_.elapsed_time(b) for _, m_, b in ev)
    ms = allreduce_max(ev[0][0].elapsed_time(ev[-1][2]) / args.steps, dist, world, dev)
    value = B * world / (ms / 1e3)
    # attainable roofline of the op sequence: each op at min(tensor, HBM) speed
    m = B * t * h * w
    ops = block_ops(m)
    P, BW = peaks["bf16_tflops"] * 1e12, peaks["hbm_gbs"] * 1e9
    floor = [(n_, max(f / P, by / BW)) for n_, f, by in ops]
    fwd_floor = sum(tt for n_, tt in floor if n_.startswith("fwd"))
    bwd_floor = sum(tt for n_, tt in floor if n_.startswith("bwd"))
    flops = sum(f for _, f, _ in ops)
    # e2e: host (pinned) x and gy in, gx out, through the same C-ABI calls
    xh, gyh = x.cpu().pin_memory(), gy.cpu().pin_memory()
    gxh = torch.empty_like(xh).pin_memory()

    def e2e_step():
        xd = xh.to(dev, non_blocking=True)
        gyd = gyh.to(dev, non_blocking=True)
        yd = blk.forward(xd)
        gxd, _ = blk.backward(xd, yd, gyd)
        gxh.copy_(gxd, non_blocking=True)
        torch.cuda.current_stream(dev).synchronize()
    e2e_step()
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    n_e2e = max(3, min(args.steps, 5))
    for _ in range(n_e2e):
        e2e_step()
    e2e_s = allreduce_max((time.perf_counter() - t0) / n_e2e, dist, world, dev)
    if rank == 0:
        cpu = None
        if not args.no_cpu_baseline and world == 1:
            try:
                r = cpu_reference_block()
                cpu = {k: r[k] for k in ("value", "unit", "cores", "kind", "sample")}
            except Exception as exc:
                cpu = {"value": None, "unit": "clips/s", "cores": 0, "kind": "reference",
                       "sample": f"unavailable: {exc}"}
        line = {"metric": "TSM bottleneck block fwd+bwd clips/sec", "value": value,
                "unit": "clips/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "bf16", "data": "synthetic N(0,1) clips, "
                "init_conv-distributed weights", "config": block_config(B, world),
                "fwd_us": fwd_ms * 1e3, "bwd_us": bwd_ms * 1e3,
                "roofline": {"bound": "attainable min(tensor, HBM) per op",
                             "achieved": flops / (ms / 1e3) / 1e12, "unit": "TFLOP/s",
                             "attainable_us": (fwd_floor + bwd_floor) * 1e6,
                             "attainable_fwd_us": fwd_floor * 1e6,
                             "attainable_bwd_us": bwd_floor * 1e6,
                             "frac": (fwd_floor + bwd_floor) / (ms / 1e3),
                             "frac_fwd": fwd_floor / (fwd_ms / 1e3),
                             "frac_bwd": bwd_floor / (bwd_ms / 1e3),
                             "peak": {"hbm_gbs": peaks["hbm_gbs"],
                                      "bf16_tflops": peaks["bf16_tflops"],
                                      "source": peaks["source"] + " (burst: timed alone)"},
                             "ops": [{"op": n_, "gflop": f / 1e9, "mb": by / 1e6,
                                      "floor_us": max(f / P, by / BW) * 1e6}
                                     for n_, f, by in ops],
                             "traffic": None},
                "cpu_baseline": cpu,
                "e2e": {"value": B * world / e2e_s, "unit": "clips/s",
                        "h2d_bytes_per_step": 2 * x.numel() * 2,
                        "d2h_bytes_per_step": x.numel() * 2,
                        "path": "Bottleneck.forward/backward (C ABI tsm_block_fwd/bwd) with x "
                                "and gy copied from pinned host memory and gx read back"},
                "gpu_launches": launches // args.steps * args.steps, "clocks": clk.summary()}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def cpu_reference_block(ref=None):
    """The reference's own op sequence for one unit (vref_block: run_unit +
    the unit's part of loss_gradients, fp64, OpenMP) at N=1, C=256, T=8,
    56x56."""
    import numpy as np
    from oracle.oracle import Reference
    ref = ref or Reference()
    c, t, h, w = BLOCK["c"], BLOCK["t"], BLOCK["h"], BLOCK["w"]
    x = ref.random_normal((1, t, c, h, w), 1)
    wd = c // 4
    shapes = [(wd, c, 1, 1, 1), (wd, wd, 1, 3, 3), (c, wd, 1, 1, 1)]
    ws = []
    for i, shp in enumerate(shapes):
        fan = shp[1] * shp[3] * shp[4]
        ws += [ref.random_normal(shp, 100 + 2 * i, (2.0 / fan) ** 0.5),
               ref.random_normal((shp[0], 1, 1, 1, 1), 101 + 2 * i, 0.1).reshape(-1)]
    ws += [None, None]
    gy = ref.random_normal((1, t, c, h, w), 2)
    t0 = time.perf_counter()
    ref.block(x, ws, c, 1, (1, 8), gy=gy)
    secs = time.perf_counter() - t0
    cores = int(os.environ.get("OMP_NUM_THREADS", os.cpu_count() or 1))
    return {"value": 1.0 / secs, "unit": "clips/s", "cores": cores, "kind": "reference",
            "seconds": secs,
            "sample": f"reference op sequence of one unit (run_unit + loss_gradients' unit "
                      f"backward, fp64, OpenMP {cores} threads) on 1 clip (1,8,256,56,56): "
                      f"{secs:.2f} s"}


def run_reference_block(args):
    B = args.batch or 8
    from oracle.oracle import Reference
    ref = Reference()
    for _ in range(args.warmup):
        cpu_reference_block(ref)
    secs = [cpu_reference_block(ref)["seconds"] for _ in range(args.steps)]
    ms = statistics.mean(secs) * 1e3
    value = 1.0 / (ms / 1e3)
    cores = int(os.environ.get("OMP_NUM_THREADS", os.cpu_count() or 1))
    sample = ("reference op sequence of one unit (fp64, OpenMP) on 1 clip per step of the "
              f"configured {B}-clip batch")
    line = {"impl": "reference", "metric": "TSM bottleneck block fwd+bwd clips/sec",
            "value": value, "unit": "clips/s", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": block_config(B, 1),
            "cpu_baseline": {"value": value, "unit": "clips/s", "cores": cores,
                             "kind": "reference", "sample": sample},
            "e2e": {"value": value, "unit": "clips/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def shift_sweep(tsm, torch, dev, stream, peaks):
    """BASELINE configs[4]: C 64-2048 x T 8/16 x fp32/bf16 at N=8, 56x56; L2
    flushed (256 MB write) before every timed launch."""
    out = []
    cfg = tsm.ShiftConfig.fold_div(8)
    flush = torch.empty(64 * 1024 * 1024, device=dev)
    for dtype, elt in ((torch.float32, 4), (torch.bfloat16, 2)):
        for t in SWEEP_T:
            for c in SWEEP_C:
                shape = (8, t, c, 56, 56)
                x = torch.empty(shape, device=dev, dtype=dtype).normal_()
                y = torch.empty_like(x)
                for _ in range(3):
                    tsm.temporal_shift(x, cfg, out=y)
                ts = []
                for _ in range(5):
                    flush.fill_(0.0)
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record(stream)
                    tsm.temporal_shift(x, cfg, out=y)
                    e1.record(stream)
                    torch.cuda.synchronize()
                    ts.append(e0.elapsed_time(e1) / 1e3)
                sec = statistics.median(ts)
                gbs = shift_bytes(shape, elt) / sec / 1e9
                out.append({"C": c, "T": t, "dtype": str(dtype).split(".")[-1],
                            "GBps": round(gbs, 1), "frac": round(gbs / peaks["hbm_gbs"], 3),
                            "us": round(sec * 1e6, 1)})
                del x, y
    torch.cuda.empty_cache()
    return out


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    elif args.workload == "train":
        run_train(args)
    elif args.workload == "block":
        run_block(args)
    else:
        run_shift(args)


if __name__ == "__main__":
    main()
