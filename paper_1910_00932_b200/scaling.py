"""The reference's cluster performance model (sim.hpp / sim.cpp), restated
and calibrated for one B200 NVL8 node, plus an overlap-aware step time.

SURVEY §8(f) f4: lets the reference's own model predict / explain the
measured 1 -> N GPU scaling of the data-parallel step.  GPUs play the role of
the reference's "nodes" (as in its observed-scalability CSV), one GPU each.

Reference semantics kept exactly (pinned against oracle/_ref in
tests/test_scaling.py): ``compute_time`` (sim.cpp:104-111), ``io_time``
(113-118), ``comm_time`` Simple / Ring (120-130), ``step_time`` with
compute/IO overlap and NO communication overlap (132-144),
``observed_scalability`` (195-215), ``load_timings_csv`` (217-240).

Added (not in the reference): ``step_time_overlapped`` — this framework
launches each gradient bucket on a communication stream as soon as its last
gradient is final (network.cu dp step), so only the last bucket's allreduce
is exposed after the backward pass."""
from __future__ import annotations

import json
from dataclasses import dataclass, replace
from pathlib import Path

from ._lib import ValidationError

# build_tsm8f per clip (cost_test.cpp:68-72): MACs 32,697,909,248 -> FLOPs x2
TSM8F_FLOPS = 2 * 32_697_909_248
TSM8F_PARAMS = 24_301_072
TSM8F_INPUT_BYTES = 8 * 3 * 224 * 224  # decoded uint8 frames per clip


@dataclass(frozen=True)
class ClusterProfile:
    """sim.hpp:12-21 (same fields, same defaults)."""
    nodes: int = 1
    gpus_per_node: int = 6
    peak_flops_per_gpu: float = 0.0
    utilization: float = 0.0
    disk_bandwidth_per_node: float = 0.0
    net_latency: float = 0.0
    net_bandwidth: float = 0.0
    bytes_per_param: float = 4.0

    def as_list(self):
        return [self.nodes, self.gpus_per_node, self.peak_flops_per_gpu, self.utilization,
                self.disk_bandwidth_per_node, self.net_latency, self.net_bandwidth,
                self.bytes_per_param]


def validate_profile(p: ClusterProfile) -> None:
    """sim.cpp:16-30."""
    def positive(v, what):
        if not v > 0.0:
            raise ValidationError(f"profile {what} must be > 0")
    if p.nodes < 1:
        raise ValidationError("profile nodes must be >= 1")
    if p.gpus_per_node < 1:
        raise ValidationError("profile gpus_per_node must be >= 1")
    positive(p.peak_flops_per_gpu, "peak_flops_per_gpu")
    if not (p.utilization > 0.0) or p.utilization > 1.0:
        raise ValidationError("profile utilization must be in (0, 1]")
    positive(p.disk_bandwidth_per_node, "disk_bandwidth_per_node")
    if p.net_latency < 0.0:
        raise ValidationError("profile net_latency must be >= 0")
    positive(p.net_bandwidth, "net_bandwidth")
    positive(p.bytes_per_param, "bytes_per_param")


def compute_time(flops_per_clip, p: ClusterProfile, per_gpu_clips, mult=3.0):
    if per_gpu_clips < 1:
        raise ValidationError("per-GPU batch must be >= 1")
    if mult <= 0.0:
        raise ValidationError("flop multiplier must be > 0")
    return per_gpu_clips * float(flops_per_clip) * mult / (p.peak_flops_per_gpu * p.utilization)


def io_time(input_bytes_per_clip, p: ClusterProfile, clips_per_node):
    if clips_per_node < 0:
        raise ValidationError("clips per node must be >= 0")
    return clips_per_node * float(input_bytes_per_clip) / p.disk_bandwidth_per_node


def comm_time(params, p: ClusterProfile, ring=True):
    if params < 0:
        raise ValidationError("params must be >= 0")
    if p.nodes == 1:
        return 0.0
    n = float(p.nodes)
    size = float(params) * p.bytes_per_param
    if not ring:
        return p.net_latency + size / p.net_bandwidth
    return 2.0 * (n - 1.0) * p.net_latency + (2.0 * (n - 1.0) / n) * size / p.net_bandwidth


@dataclass
class StepTime:
    t_compute: float
    t_io: float
    t_comm: float
    t_step: float
    bottleneck: str


def step_time(p: ClusterProfile, per_gpu_batch=64, mult=3.0, ring=True,
              flops=TSM8F_FLOPS, params=TSM8F_PARAMS, input_bytes=TSM8F_INPUT_BYTES):
    """sim.cpp:132-144: max(compute, io) + comm (communication not overlapped)."""
    validate_profile(p)
    tc = compute_time(flops, p, per_gpu_batch, mult)
    ti = io_time(input_bytes, p, per_gpu_batch * p.gpus_per_node)
    tm = comm_time(params, p, ring)
    return StepTime(tc, ti, tm, max(tc, ti) + tm, "io" if ti > tc else "compute")


def step_time_overlapped(p: ClusterProfile, bucket_bytes=25 << 20, per_gpu_batch=64, mult=3.0,
                         flops=TSM8F_FLOPS, params=TSM8F_PARAMS, input_bytes=TSM8F_INPUT_BYTES):
    """Bucketed allreduce overlapped with backward: the buckets before the
    last run under the remaining backward compute (they are exposed only if
    the ring is slower than backward), the last one (the stem / first layers,
    the smallest tail, at most `bucket_bytes`) is not."""
    st = step_time(p, per_gpu_batch, mult, True, flops, params, input_bytes)
    if p.nodes == 1:
        return st
    last = min(float(bucket_bytes), params * p.bytes_per_param)
    tail = comm_time(last / p.bytes_per_param, p, True)
    body = st.t_comm - tail
    bwd = st.t_compute * (mult - 1.0) / mult  # backward share of the step
    exposed = tail + max(0.0, body - bwd)
    return StepTime(st.t_compute, st.t_io, st.t_comm, max(st.t_compute, st.t_io) + exposed,
                    st.bottleneck)


def observed_scalability(timings):
    """sim.cpp:195-215: baseline / (p * time(p)); needs a p = 1 row."""
    base = None
    for nodes, secs in timings:
        if nodes < 1:
            raise ValidationError("node counts must be >= 1")
        if not secs > 0.0:
            raise ValidationError("wall times must be > 0")
        if nodes == 1:
            base = secs
    if base is None:
        raise ValidationError("timings need a 1-node row to define the scalability baseline")
    return [(nodes, base / (nodes * secs)) for nodes, secs in timings]


def load_timings_csv(path):
    """sim.cpp:217-240: header ``nodes,wall_seconds``."""
    try:
        lines = Path(path).read_text().splitlines()
    except OSError:
        raise ValidationError(f"cannot open timings '{path}'") from None
    if not lines or lines[0] != "nodes,wall_seconds":
        raise ValidationError(f"timings '{path}' must start with header nodes,wall_seconds")
    out = []
    for line in lines[1:]:
        if not line:
            continue
        parts = line.split(",")
        if len(parts) != 2:
            raise ValidationError(f"timings '{path}': bad row '{line}'")
        try:
            out.append((int(parts[0]), float(parts[1])))
        except ValueError:
            raise ValidationError(f"timings '{path}': bad row '{line}'") from None
    return out


def b200_profile(nodes=1, utilization=0.36, net_latency=8e-6, net_bandwidth=700e9,
                 peaks_path=None) -> ClusterProfile:
    """One B200 per "node" over NVLink 5 / NVSwitch.  peak = the measured
    sustained dense bf16 rate (MEASURED_PEAKS.json), utilization = the
    measured single-GPU step's tensor fraction (bench ``step_tensor.frac``),
    net_bandwidth = NCCL allreduce bus bandwidth.  Disk: synthetic in-HBM
    input (the step reads no disk), modelled as never the bottleneck."""
    peak = 1419.9e12
    path = Path(peaks_path) if peaks_path else Path(__file__).resolve().parents[1] / "MEASURED_PEAKS.json"
    if path.exists():
        try:
            d = json.loads(path.read_text())
            for k in ("bf16_tflops_sustained", "bf16_tflops"):
                if k in d:
                    peak = float(d[k]) * 1e12
                    break
        except (ValueError, TypeError):
            pass
    return ClusterProfile(nodes=nodes, gpus_per_node=1, peak_flops_per_gpu=peak,
                          utilization=utilization, disk_bandwidth_per_node=1e15,
                          net_latency=net_latency, net_bandwidth=net_bandwidth,
                          bytes_per_param=4.0)


def with_nodes(p: ClusterProfile, nodes: int) -> ClusterProfile:
    return replace(p, nodes=nodes)
