"""The residual-shift TSM bottleneck unit — host-side mirror of the
reference's unit (``expand_layer`` arch.cpp:278-323 executed by
``Network::run_unit`` net.cpp:85-126 and reversed by ``loss_gradients``
net.cpp:184-248) over the C ABI ``tsm_block_fwd`` / ``tsm_block_bwd``.

Parameters are fp32 CUDA tensors in the GEMM layout [c_out][kh][kw][c_in];
``from_reference`` / ``to_reference`` convert from/to the reference layout
(c_out, c_in, kt, kh, kw) of ``ConvWeights`` (kernels.hpp:34-45).
Activations are NTHWC bf16."""
from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _lib
from .shift import ShiftConfig, split

NAMES = ("w1", "b1", "w2", "b2", "w3", "b3", "wp", "bp")


def ref_to_gemm(w):
    """(c_out, c_in, kt, kh, kw) -> (c_out, kh, kw, c_in), kt = 1."""
    w = torch.as_tensor(w)
    assert w.dim() == 5 and w.shape[2] == 1
    return w[:, :, 0].permute(0, 2, 3, 1).contiguous()


def gemm_to_ref(w):
    return w.permute(0, 3, 1, 2).unsqueeze(2).contiguous()


class Bottleneck:
    def __init__(self, c_in, c_out, stride=1, shift: ShiftConfig | None = ShiftConfig(),
                 device="cuda"):
        if c_out % 4:
            raise _lib.ValidationError(
                f"bottleneck channels_out {c_out} is not a positive multiple of 4")
        self.c_in, self.c_out, self.stride = c_in, c_out, stride
        self.width = c_out // 4
        self.shift = shift
        self.fold = split(shift, c_in) if shift is not None else (0, 0)
        self.has_proj = stride != 1 or c_in != c_out
        self.device = torch.device(device)
        self.params: dict[str, torch.Tensor | None] = {k: None for k in NAMES}
        self._ws = None
        self._ws_key = None

    # -- parameters ---------------------------------------------------------
    def shapes(self):
        w, ci, co = self.width, self.c_in, self.c_out
        s = {"w1": (w, 1, 1, ci), "b1": (w,), "w2": (w, 3, 3, w), "b2": (w,),
             "w3": (co, 1, 1, w), "b3": (co,)}
        if self.has_proj:
            s.update({"wp": (co, 1, 1, ci), "bp": (co,)})
        return s

    def load_reference(self, ws):
        """ws = [w1,b1,w2,b2,w3,b3,wp,bp] in the reference layout (numpy/torch)."""
        for name, w in zip(NAMES, ws):
            if w is None:
                continue
            t = torch.as_tensor(np.asarray(w), dtype=torch.float32)
            if name.startswith("w"):
                t = ref_to_gemm(t)
            self.params[name] = t.to(self.device).contiguous()
        for k, s in self.shapes().items():
            if self.params[k] is None or tuple(self.params[k].shape) != s:
                raise _lib.ValidationError(f"block parameter {k}: expected {s}")
        return self

    # -- execution ----------------------------------------------------------
    def _check_device(self, *ts):
        if self.device.index is None:  # "cuda": bind to the current device on first use
            self.device = torch.device("cuda", torch.cuda.current_device())
        for t in ts:
            if not t.is_cuda or t.device != self.device:
                raise ValueError(f"Bottleneck: tensor on {t.device}, block on {self.device}")

    def desc(self, x_shape):
        n, t, h, w, c = x_shape
        if c != self.c_in:
            raise _lib.ValidationError(f"block expects {self.c_in} input channels, tensor has {c}")
        return _lib.BlockDesc(n, t, h, w, self.c_in, self.c_out, self.stride, self.fold[0],
                              self.fold[1])

    def _ptrs(self, d):
        return _lib.BlockPtrs(*[(d[k].data_ptr() if d.get(k) is not None else None) for k in NAMES])

    def _workspace(self, d):
        key = (d.n, d.t, d.h, d.w)
        if self._ws_key != key:
            nbytes = _lib.lib.tsm_block_workspace_bytes(C.byref(d))
            self._ws = torch.empty(nbytes, device=self.device, dtype=torch.uint8)
            self._ws_key = key
        return self._ws

    def out_shape(self, x_shape):
        n, t, h, w, _ = x_shape
        return (n, t, (h - 1) // self.stride + 1, (w - 1) // self.stride + 1, self.c_out)

    def forward(self, x):
        self._check_device(x)
        d = self.desc(x.shape)
        y = torch.empty(self.out_shape(x.shape), device=x.device, dtype=torch.bfloat16)
        ws = self._workspace(d)
        with torch.cuda.device(x.device):
            stream = torch.cuda.current_stream(x.device).cuda_stream
            _lib.check(_lib.lib.tsm_block_fwd(C.byref(d), C.byref(self._ptrs(self.params)),
                                              x.data_ptr(), y.data_ptr(), ws.data_ptr(), stream))
        return y

    def backward(self, x, y, gy):
        """Gradients w.r.t. x (NTHWC bf16) and every parameter (fp32, GEMM
        layout).  Must follow ``forward(x)`` (the workspace holds its saved
        activations)."""
        self._check_device(x, y, gy)
        d = self.desc(x.shape)
        ws = self._workspace(d)
        gx = torch.empty_like(x)
        grads = {k: torch.empty(s, device=x.device, dtype=torch.float32)
                 for k, s in self.shapes().items()}
        with torch.cuda.device(x.device):
            stream = torch.cuda.current_stream(x.device).cuda_stream
            _lib.check(_lib.lib.tsm_block_bwd(C.byref(d), C.byref(self._ptrs(self.params)),
                                              x.data_ptr(), y.data_ptr(), gy.data_ptr(),
                                              gx.data_ptr(), C.byref(self._ptrs(grads)),
                                              ws.data_ptr(), stream))
        return gx, grads
