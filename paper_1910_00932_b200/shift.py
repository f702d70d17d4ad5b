"""Temporal shift — host-side mirror of the reference operator API.

Same names, argument meaning and error behaviour as the reference
(include/vidperf/kernels.hpp:11-26, src/kernels.cpp:82-157,
include/vidperf/rational.hpp:12-33): ``ShiftConfig`` holds two exact
``Rational`` fractions, ``validate_shift`` raises ``ValidationError`` unless
the split is integral, ``temporal_shift`` / ``temporal_shift_adjoint`` return
a NEW tensor (value semantics; never in place).  Tensors are torch CUDA
tensors in the reference layout [N][T][C][H][W]; the work runs in
libtsm_b200.so on the current CUDA stream.  CPU tensors are rejected: there
is no CPU path in the product.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from math import gcd

import torch

from . import _lib
from ._lib import ValidationError

_DTYPES = {
    torch.float32: _lib.TSM_F32,
    torch.bfloat16: _lib.TSM_BF16,
    torch.float64: _lib.TSM_F64,
    torch.float16: _lib.TSM_F16,
}


@dataclass(frozen=True)
class Rational:
    """Exact fraction, normalised with den > 0 (rational.cpp:10-23)."""

    num: int = 0
    den: int = 1

    def __post_init__(self):
        num, den = int(self.num), int(self.den)
        if den == 0:
            raise ValidationError("rational with zero denominator")
        if den < 0:
            num, den = -num, -den
        if num == 0:
            den = 1
        else:
            g = gcd(abs(num), den)
            num, den = num // g, den // g
        object.__setattr__(self, "num", num)
        object.__setattr__(self, "den", den)

    def is_zero(self) -> bool:
        return self.num == 0

    def __str__(self):
        return f"{self.num}/{self.den}"


def parse_rational(text: str) -> Rational:
    """"p/q" or a bare integer "p" (rational.cpp:39-48)."""
    try:
        if "/" not in text:
            return Rational(int(text), 1)
        p, q = text.split("/", 1)
        return Rational(int(p), int(q))
    except ValueError as e:
        raise ValidationError(f"bad rational '{text}'") from e


@dataclass(frozen=True)
class ShiftConfig:
    """Channels [0,F) read t-1, [F,F+B) read t+1 (kernels.hpp:13-18)."""

    fraction_fwd: Rational = Rational(1, 8)
    fraction_bwd: Rational = Rational(1, 8)

    @staticmethod
    def symmetric(fraction: Rational) -> "ShiftConfig":
        return ShiftConfig(fraction, fraction)

    @staticmethod
    def fold_div(div: int = 8) -> "ShiftConfig":
        return ShiftConfig.symmetric(Rational(1, div))


def split(cfg: ShiftConfig, channels: int) -> tuple[int, int]:
    """(F, B) for ``channels`` or ValidationError (kernels.cpp:82-101)."""
    f, b = C.c_int64(), C.c_int64()
    _lib.check(_lib.lib.tsm_validate_shift(cfg.fraction_fwd.num, cfg.fraction_fwd.den,
                                           cfg.fraction_bwd.num, cfg.fraction_bwd.den,
                                           int(channels), C.byref(f), C.byref(b)))
    return f.value, b.value


def validate_shift(cfg: ShiftConfig, channels: int) -> None:
    """kernels.hpp:22 — raises ValidationError unless the split is integral."""
    split(cfg, channels)


def _launch(x: torch.Tensor, cfg: ShiftConfig, adjoint: bool, out: torch.Tensor | None):
    if x.dim() != 5:
        raise ValidationError(f"temporal shift expects a 5-D [N][T][C][H][W] tensor, got {x.dim()}-D")
    if not x.is_cuda:
        raise ValueError("temporal_shift: the B200 path takes CUDA tensors (no CPU fallback)")
    if x.dtype not in _DTYPES:
        raise NotImplementedError(f"temporal_shift: dtype {x.dtype} not supported")
    x = x.contiguous()
    n, t, c, h, w = x.shape
    f, b = split(cfg, c)
    y = torch.empty_like(x) if out is None else out
    if y.shape != x.shape or y.dtype != x.dtype or not y.is_contiguous():
        raise ValidationError("temporal_shift: out must be a contiguous tensor like x")
    if y.device != x.device:
        raise ValueError(f"temporal_shift: out is on {y.device}, x on {x.device}")
    fn = _lib.lib.tsm_shift_bwd if adjoint else _lib.lib.tsm_shift_fwd
    with torch.cuda.device(x.device):
        stream = torch.cuda.current_stream(x.device).cuda_stream
        _lib.check(fn(x.data_ptr(), y.data_ptr(), n, t, c, h, w, f, b, _DTYPES[x.dtype], stream))
    return y


def temporal_shift(x: torch.Tensor, cfg: ShiftConfig = ShiftConfig(), *, out=None) -> torch.Tensor:
    """kernels.hpp:24 / kernels.cpp:97-125."""
    return _launch(x, cfg, False, out)


def temporal_shift_adjoint(y: torch.Tensor, cfg: ShiftConfig = ShiftConfig(), *, out=None) -> torch.Tensor:
    """kernels.hpp:26 / kernels.cpp:127-157."""
    return _launch(y, cfg, True, out)


def temporal_shift_host(x, cfg: ShiftConfig = ShiftConfig(), adjoint: bool = False, out=None):
    """Host-buffer path through the C ABI (``tsm_shift_host``): a numpy array or
    CPU torch tensor in, a new one out; H2D copy, kernel, D2H copy inside."""
    import numpy as np

    is_torch = isinstance(x, torch.Tensor)
    arr = x if is_torch else np.ascontiguousarray(x)
    if is_torch:
        if arr.is_cuda:
            raise ValueError("temporal_shift_host takes host memory")
        arr = arr.contiguous()
        if arr.dtype not in _DTYPES:
            raise NotImplementedError(f"temporal_shift_host: dtype {arr.dtype} not supported")
        dt = _DTYPES[arr.dtype]
        y = torch.empty_like(arr) if out is None else out
        if not isinstance(y, torch.Tensor) or y.is_cuda or y.shape != arr.shape \
                or y.dtype != arr.dtype or not y.is_contiguous():
            raise ValidationError("temporal_shift_host: out must be a contiguous host tensor "
                                  "like x")
        xp, yp = arr.data_ptr(), y.data_ptr()
    else:
        npmap = {np.dtype(np.float32): _lib.TSM_F32, np.dtype(np.float64): _lib.TSM_F64,
                 np.dtype(np.float16): _lib.TSM_F16}
        if arr.dtype not in npmap:
            raise NotImplementedError(f"temporal_shift_host: dtype {arr.dtype} not supported")
        dt = npmap[arr.dtype]
        y = np.empty_like(arr) if out is None else out
        if not isinstance(y, np.ndarray) or y.shape != arr.shape or y.dtype != arr.dtype \
                or not y.flags.c_contiguous or not y.flags.writeable:
            raise ValidationError("temporal_shift_host: out must be a contiguous writable "
                                  "array like x")
        xp, yp = arr.ctypes.data, y.ctypes.data
    n, t, c, h, w = arr.shape
    f, b = split(cfg, c)
    _lib.check(_lib.lib.tsm_shift_host(xp, yp, n, t, c, h, w, f, b, dt, int(adjoint)))
    return y
