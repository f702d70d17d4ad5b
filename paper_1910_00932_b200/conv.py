"""Torch-tensor wrappers over the tcgen05 conv entry points of the C ABI
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


def out_hw(h, w, k, stride):
    return (h + 2 * (k // 2) - k) // stride + 1, (w + 2 * (k // 2) - k) // stride + 1


def conv_fwd(x, w, bias, *, k=1, stride=1, fold=(0, 0), relu=False, residual=None, out=None):
    """y = act(conv_k(shift(x)) + bias (+ residual)); x NTHWC bf16, w [c_out][k][k][c_in]."""
    n, t, h, wd, cin = x.shape
    cout = w.shape[0]
    for a, nm in ((x, "x"), (w, "w"), (residual, "residual")):
        _need(a, torch.bfloat16, nm)
    _need(bias, torch.float32, "bias")
    ho, wo = out_hw(h, wd, k, stride)
    y = torch.empty((n, t, ho, wo, cout), device=x.device, dtype=torch.bfloat16) if out is None else out
    _lib.check(_lib.lib.tsm_conv_fwd(_ptr(x), _ptr(w), _ptr(bias), _ptr(residual), _ptr(y),
                                     n, t, h, wd, cin, cout, k, stride, fold[0], fold[1],
                                     int(relu), _stream(x)))
    return y


def conv1x1_fwd(x, w, bias, *, fold=(0, 0), relu=False, residual=None, out=None):
    return conv_fwd(x, w, bias, k=1, stride=1, fold=fold, relu=relu, residual=residual, out=out)


def conv_dgrad(dy, wt, x_shape, *, k=1, stride=1, fold=(0, 0), residual=None, mask=None,
               out=None):
    """dx = mask? (shift_adjoint(dgrad(dy)) + residual); wt = dgrad operand [c_in][k][k][c_out]."""
    n, t, h, wd, cin = x_shape
    cout = dy.shape[-1]
    for a, nm in ((dy, "dy"), (wt, "wt"), (residual, "residual"), (mask, "mask")):
        _need(a, torch.bfloat16, nm)
    dx = torch.empty(x_shape, device=dy.device, dtype=torch.bfloat16) if out is None else out
    scratch = None
    ho, wo = out_hw(h, wd, k, stride)
    if k > 1 and stride > 1 and not (k == 3 and h == 2 * ho and wd == 2 * wo):
        scratch = torch.empty((n, t, h, wd, cout), device=dy.device, dtype=torch.bfloat16)
    _lib.check(_lib.lib.tsm_conv_dgrad(_ptr(dy), _ptr(wt), _ptr(residual), _ptr(mask), _ptr(dx),
                                       _ptr(scratch), n, t, h, wd, cin, cout, k, stride,
                                       fold[0], fold[1], _stream(dy)))
    return dx


def conv_wgrad(x, dy, *, k=1, stride=1, fold=(0, 0), out=None, bias_grad=False):
    """dw fp32 [c_out][k][k][c_in] = sum_p dy[p] (x) im2col(shift(x))[p]
    (and, with bias_grad, db = sum_p dy[p] from the same pass)."""
    n, t, h, wd, cin = x.shape
    cout = dy.shape[-1]
    _need(x, torch.bfloat16, "x")
    _need(dy, torch.bfloat16, "dy")
    dw = torch.empty((cout, k, k, cin), device=x.device, dtype=torch.float32) if out is None else out
    db = torch.empty(cout, device=x.device, dtype=torch.float32) if bias_grad else None
    nb = _lib.lib.tsm_conv_wgrad_workspace_bytes(n, t, h, wd, cin, cout, k, stride)
    ws = torch.empty(max(nb, 16) // 4 + 4, device=x.device, dtype=torch.float32)
    _lib.check(_lib.lib.tsm_conv_wgrad(_ptr(x), _ptr(dy), _ptr(dw), _ptr(db), _ptr(ws), n, t, h,
                                       wd, cin, cout, k, stride, fold[0], fold[1], _stream(x)))
    return (dw, db) if bias_grad else dw


def weights_to_bf16(w, *, k_pad=None, dgrad=True):
    """fp32 [c_out][k][k][c_in] -> (bf16 forward [c_out][k_pad], bf16 dgrad [c_in][k][k][c_out])."""
    cout, k, _, cin = w.shape
    k_pad = k * k * cin if k_pad is None else k_pad
    wf = torch.empty((cout, k_pad), device=w.device, dtype=torch.bfloat16)
    wd = torch.empty((cin, k, k, cout), device=w.device, dtype=torch.bfloat16) if dgrad else None
    _lib.check(_lib.lib.tsm_weights_to_bf16(_ptr(w), _ptr(wf), _ptr(wd), cout, cin, k, k_pad,
                                            _stream(w)))
    return wf, wd


def bias_grad(g):
    c = g.shape[-1]
    rows = g.numel() // c
    db = torch.empty(c, device=g.device, dtype=torch.float32)
    ws = torch.empty(_lib.lib.tsm_bias_grad_workspace_bytes(rows, c) // 4 + 4, device=g.device)
    _lib.check(_lib.lib.tsm_bias_grad(_ptr(g), _ptr(db), _ptr(ws), rows, c, _stream(g)))
    return db


_DT = {torch.float32: _lib.TSM_F32, torch.float64: _lib.TSM_F64, torch.bfloat16: _lib.TSM_BF16}


def to_nthwc(x, c_pad=None):
    """[N][T][C][H][W] (f32/f64/bf16) -> [N][T][H][W][c_pad] bf16."""
    n, t, c, h, w = x.shape
    c_pad = c if c_pad is None else c_pad
    x = x.contiguous()
    y = torch.empty((n, t, h, w, c_pad), device=x.device, dtype=torch.bfloat16)
    _lib.check(_lib.lib.tsm_layout_to_nthwc(_ptr(x), _DT[x.dtype], _ptr(y), n * t, c, h, w, c_pad,
                                            _stream(x)))
    return y


def to_ntchw(x, dtype=torch.float32):
    n, t, h, w, c = x.shape
    y = torch.empty((n, t, c, h, w), device=x.device, dtype=dtype)
    _lib.check(_lib.lib.tsm_layout_to_ntchw(_ptr(x), _ptr(y), _DT[dtype], n * t, c, h, w,
                                            _stream(x)))
    return y


def maxpool_fwd(x):
    """Stem max pool 1x3x3 / s2 / pad 1 on NTHWC bf16 [N][T][H][W][C]; returns
    (y, argmax bytes) (max_pool_forward kernels.cpp:353-390: first max wins)."""
    n, t, h, wd, c = x.shape
    _need(x, torch.bfloat16, "x")
    ho, wo = (h - 1) // 2 + 1, (wd - 1) // 2 + 1
    y = torch.empty((n, t, ho, wo, c), device=x.device, dtype=torch.bfloat16)
    arg = torch.empty((n, t, ho, wo, c), device=x.device, dtype=torch.uint8)
    _lib.check(_lib.lib.tsm_maxpool_fwd(_ptr(x), _ptr(y), _ptr(arg), n * t, h, wd, c,
                                        _stream(x)))
    return y, arg


def maxpool_bwd(gy, arg, x_shape):
    """Gradient routed to the recorded argmax (max_pool_backward kernels.cpp:392-455)."""
    n, t, h, wd, c = x_shape
    _need(gy, torch.bfloat16, "gy")
    gx = torch.empty(x_shape, device=gy.device, dtype=torch.bfloat16)
    _lib.check(_lib.lib.tsm_maxpool_bwd(_ptr(gy), _ptr(arg), _ptr(gx), n * t, h, wd, c,
                                        _stream(gy)))
    return gx
