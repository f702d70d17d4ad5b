"""B200-native Temporal Shift Module hot path (arXiv 1910.00932).

A drop-in for the reference library ``vidperf``'s TSM path: the temporal
shift operator and its adjoint, the residual-shift bottleneck block, and the
TSM-ResNet-50 data-parallel training step.  All compute runs in
``libtsm_b200.so`` (hand-written sm_100a CUDA behind the C ABI in
``include/tsm_b200.h``); this package is the host-side mirror of the
reference operator API.  PyTorch supplies device memory, streams and
``torch.distributed`` plumbing only.
"""
from ._lib import TsmError, ValidationError, launch_count  # noqa: F401
from .shift import (  # noqa: F401
    Rational,
    ShiftConfig,
    parse_rational,
    split,
    temporal_shift,
    temporal_shift_adjoint,
    temporal_shift_host,
    validate_shift,
)

from . import conv, network  # noqa: E402,F401
from .block import Bottleneck  # noqa: E402,F401
from .network import TSMNet  # noqa: E402,F401

__all__ = [
    "Bottleneck", "TSMNet", "conv", "network",
    "Rational", "ShiftConfig", "ValidationError", "TsmError", "parse_rational", "split",
    "validate_shift", "temporal_shift", "temporal_shift_adjoint", "temporal_shift_host",
    "launch_count",
]
