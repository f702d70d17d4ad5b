"""Thin torch-tensor wrappers over the tcgen05 conv entry points of the C ABI
(include/tsm_b200.h).  Activations are NTHWC bf16 ([N][T][H][W][C]); weights
bf16 [c_out][kh][kw][c_in]; biases fp32."""
from __future__ import annotations

import torch

from . import _lib


def _ptr(t):
    return 0 if t is None else t.data_ptr()


def _stream(t):
    return torch.cuda.current_stream(t.device).cuda_stream


def _need(t, dtype, name):
    if t is None:
        return
    if not t.is_cuda or t.dtype != dtype or not t.is_contiguous():
        raise ValueError(f"{name}: expected a contiguous CUDA {dtype} tensor")


def conv1x1_fwd(x, w, bias, *, fold=(0, 0), relu=False, residual=None, out=None):
    """y = act(conv1x1(shift(x)) + bias (+ residual)); x NTHWC bf16, w [c_out][c_in]."""
    n, t, h, wd, cin = x.shape
    cout = w.shape[0]
    _need(x, torch.bfloat16, "x")
    _need(w, torch.bfloat16, "w")
    _need(bias, torch.float32, "bias")
    _need(residual, torch.bfloat16, "residual")
    y = torch.empty((n, t, h, wd, cout), device=x.device, dtype=torch.bfloat16) if out is None else out
    _lib.check(_lib.lib.tsm_conv1x1_fwd(_ptr(x), _ptr(w), _ptr(bias), _ptr(residual), _ptr(y),
                                        n, t, h, wd, cin, cout, fold[0], fold[1], int(relu),
                                        _stream(x)))
    return y
