"""TSM-ResNet-50 8-frame network + data-parallel training step — host-side
mirror of ``vidperf::Network`` over ``build_tsm8f()`` (net.hpp:15-54,
arch.cpp:140-161) on the C ABI ``tsm_net_*`` (include/tsm_b200.h).

    net = TSMNet(batch=64)              # one per GPU
    net.init_random(seed) | net.load_reference(flat_params)
    net.dp_init()                       # under torch.distributed (NCCL)
    loss = net.train_step(x, lr=...)    # x: [N][8][3][224][224] CUDA tensor

The parameter vector is the reference's flat order (net.cpp:63-75);
``load_reference`` / ``grads_reference`` convert from/to the reference tensor
layout (c_out, c_in, kt, kh, kw)."""
from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _lib
from .shift import ShiftConfig

_i64 = C.c_int64


class NetDesc(C.Structure):
    _fields_ = [("batch", _i64), ("frames", _i64), ("height", _i64), ("width", _i64),
                ("classes", _i64), ("shift_num", _i64), ("shift_den", _i64), ("arch", _i64)]


# network presets (include/tsm_b200.h TSM_ARCH_*; arch.cpp:140-161, 220-233)
ARCHS = {"tsm8f": (0, 3), "micro-tsm": (1, 8)}  # name -> (id, input channels)


class ParamInfo(C.Structure):
    _fields_ = [("offset", _i64), ("numel", _i64), ("dims", _i64 * 4), ("ci_ref", _i64),
                ("is_bias", C.c_int32), ("name", C.c_char * 48)]


class Sgd(C.Structure):
    _fields_ = [("enabled", C.c_int32), ("lr", C.c_float), ("momentum", C.c_float),
                ("weight_decay", C.c_float), ("grad_scale", C.c_float)]


L = _lib.lib
L.tsm_net_create.argtypes = [C.POINTER(NetDesc), C.POINTER(C.c_void_p)]
L.tsm_net_create.restype = C.c_int
L.tsm_net_destroy.argtypes = [C.c_void_p]
L.tsm_net_param_count.argtypes = [C.c_void_p]
L.tsm_net_param_count.restype = _i64
L.tsm_net_param_tensors.argtypes = [C.c_void_p]
L.tsm_net_param_tensors.restype = _i64
L.tsm_net_param_info.argtypes = [C.c_void_p, _i64, C.POINTER(ParamInfo)]
L.tsm_net_param_info.restype = C.c_int
for _f in (L.tsm_net_params, L.tsm_net_grads, L.tsm_net_loss, L.tsm_net_logits):
    _f.argtypes = [C.c_void_p]
    _f.restype = C.c_void_p
L.tsm_net_forward.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_void_p, C.c_void_p]
L.tsm_net_forward.restype = C.c_int
L.tsm_net_train_step.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.POINTER(Sgd), C.c_void_p]
L.tsm_net_train_step.restype = C.c_int
L.tsm_net_set_graph.argtypes = [C.c_void_p, C.c_int]
L.tsm_net_set_graph.restype = C.c_int
L.tsm_net_input_grad.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_void_p]
L.tsm_net_input_grad.restype = C.c_int
L.tsm_nccl_unique_id.argtypes = [C.c_void_p]
L.tsm_nccl_unique_id.restype = C.c_int
L.tsm_net_dp_init.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_size_t]
L.tsm_net_dp_init.restype = C.c_int

_DT = {torch.float32: _lib.TSM_F32, torch.float64: _lib.TSM_F64, torch.bfloat16: _lib.TSM_BF16}


class _CudaView:
    """Zero-copy torch view of device memory owned by libtsm_b200."""

    def __init__(self, ptr, shape, typestr):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr,
                                         "data": (int(ptr), False), "version": 3}


def _view(ptr, shape, dtype, device):
    ts = {torch.float32: "<f4"}[dtype]
    return torch.as_tensor(_CudaView(ptr, shape, ts), device=device)


class TSMNet:
    def __init__(self, batch, frames=8, height=224, width=224, classes=400,
                 shift: ShiftConfig | None = ShiftConfig(), device=None, arch="tsm8f"):
        """arch: "tsm8f" (build_tsm8f) or "micro-tsm" (build_micro_tsm: input
        (N, 4, 8, 5, 5), two 16-channel units, 4 classes in the reference)."""
        self.device = torch.device("cuda", torch.cuda.current_device()) if device is None \
            else torch.device(device)
        if arch not in ARCHS:
            raise _lib.ValidationError(f"unknown preset '{arch}'")
        self.arch = arch
        self.in_channels = ARCHS[arch][1]
        self.batch, self.frames, self.classes = batch, frames, classes
        self.height, self.width = height, width
        frac = shift.fraction_fwd if shift is not None else None
        d = NetDesc(batch, frames, height, width, classes, frac.num if frac else 0,
                    frac.den if frac else 1, ARCHS[arch][0])
        h = C.c_void_p()
        with torch.cuda.device(self.device):
            _lib.check(L.tsm_net_create(C.byref(d), C.byref(h)))
        self.h = h
        self.n_params = L.tsm_net_param_count(h)
        self.table = []
        for i in range(L.tsm_net_param_tensors(h)):
            p = ParamInfo()
            _lib.check(L.tsm_net_param_info(h, i, C.byref(p)))
            self.table.append({"name": p.name.decode(), "offset": p.offset, "numel": p.numel,
                               "dims": tuple(p.dims), "ci_ref": p.ci_ref,
                               "is_bias": bool(p.is_bias)})
        self.params = _view(L.tsm_net_params(h), (self.n_params,), torch.float32, self.device)
        self.grads = _view(L.tsm_net_grads(h), (self.n_params,), torch.float32, self.device)
        self.loss = _view(L.tsm_net_loss(h), (1,), torch.float32, self.device)
        self.logits = _view(L.tsm_net_logits(h), (batch, classes), torch.float32, self.device)
        self.world = 1

    def __del__(self):
        if getattr(self, "h", None):
            L.tsm_net_destroy(self.h)
            self.h = None

    # -- parameters -----------------------------------------------------------
    def reference_param_count(self):
        return sum(t["dims"][0] * t["dims"][1] * t["dims"][2] * t["ci_ref"] for t in self.table)

    def init_random(self, seed=0):
        """init_conv / init_fc distributions (net.cpp:14-31): weights
        N(0, sqrt(2/fan_in)), biases N(0, 0.1); padded stem channels zero."""
        g = torch.Generator(device=self.device).manual_seed(seed)
        with torch.no_grad():
            for t in self.table:
                co, kh, kw, ci = t["dims"]
                v = self.params[t["offset"]:t["offset"] + t["numel"]].view(co, kh, kw, ci)
                if t["is_bias"]:
                    v.normal_(0.0, 0.1, generator=g)
                else:
                    fan = t["ci_ref"] * kh * kw
                    v.zero_()
                    v[..., :t["ci_ref"]].normal_(0.0, (2.0 / fan) ** 0.5, generator=g)
        return self

    def load_reference(self, flat):
        """flat: the reference param_vector() (net.hpp:24), reference layout."""
        flat = np.asarray(flat, dtype=np.float64)
        if flat.size != self.reference_param_count():
            raise _lib.ValidationError(f"expected {self.reference_param_count()} parameters, "
                                       f"got {flat.size}")
        out = np.zeros(self.n_params, np.float32)
        pos = 0
        for t in self.table:
            co, kh, kw, ci = t["dims"]
            n = co * kh * kw * t["ci_ref"]
            src = flat[pos:pos + n]
            pos += n
            if t["is_bias"]:
                out[t["offset"]:t["offset"] + t["numel"]] = src
                continue
            w = src.reshape(co, t["ci_ref"], kh, kw).transpose(0, 2, 3, 1)  # kt = 1
            full = np.zeros((co, kh, kw, ci), np.float32)
            full[..., :t["ci_ref"]] = w
            out[t["offset"]:t["offset"] + t["numel"]] = full.ravel()
        with torch.no_grad():
            self.params.copy_(torch.from_numpy(out).to(self.device))
        return self

    def to_reference(self, vec):
        """Flat GEMM-layout vector (params or grads) -> reference flat order/layout."""
        v = vec.detach().double().cpu().numpy()
        out = []
        for t in self.table:
            co, kh, kw, ci = t["dims"]
            x = v[t["offset"]:t["offset"] + t["numel"]]
            if t["is_bias"]:
                out.append(x)
            else:
                out.append(x.reshape(co, kh, kw, ci)[..., :t["ci_ref"]]
                           .transpose(0, 3, 1, 2).ravel())
        return np.concatenate(out)

    def grads_reference(self):
        return self.to_reference(self.grads)

    # -- execution ------------------------------------------------------------
    def _x(self, x):
        if not x.is_cuda or x.dtype not in _DT:
            raise ValueError("TSMNet: x must be a CUDA f32/f64/bf16 tensor [N][T][C][H][W]")
        if x.device != self.device:
            raise ValueError(f"TSMNet: x is on {x.device}, the network on {self.device}")
        want = (self.batch, self.frames, self.in_channels, self.height, self.width)
        if tuple(x.shape) != want:
            raise _lib.ValidationError(f"input {tuple(x.shape)} does not match the architecture "
                                       f"{want}")
        return x.contiguous()

    def forward(self, x):
        """net.cpp:128-139; returns a copy of the logits [N][classes]."""
        x = self._x(x)
        with torch.cuda.device(self.device):
            st = torch.cuda.current_stream(self.device).cuda_stream
            _lib.check(L.tsm_net_forward(self.h, x.data_ptr(), _DT[x.dtype], None, st))
        return self.logits.clone()

    def train_step(self, x, *, lr=0.0, momentum=0.9, weight_decay=1e-4, grad_scale=None,
                   update=True):
        """Forward, sum-of-squares loss, backward, NCCL gradient allreduce
        (if dp_init), SGD update.  Returns the device loss scalar (a view)."""
        x = self._x(x)
        if grad_scale is None:
            grad_scale = 1.0 / (self.batch * self.world)
        opt = Sgd(int(update), lr, momentum, weight_decay, grad_scale)
        with torch.cuda.device(self.device):
            st = torch.cuda.current_stream(self.device).cuda_stream
            _lib.check(L.tsm_net_train_step(self.h, x.data_ptr(), _DT[x.dtype], C.byref(opt), st))
        return self.loss

    def set_graph(self, enable=True):
        """CUDA-graph replay of train_step (tsm_net_set_graph): for small,
        launch-bound batches.  Single GPU; eager under data parallelism."""
        _lib.check(L.tsm_net_set_graph(self.h, int(enable)))
        return self

    def input_grad(self, dtype=torch.float32):
        """dL/dx of the last train_step (Gradients::input, net.hpp:39), in the
        input's layout [N][T][C][H][W]."""
        gx = torch.empty((self.batch, self.frames, self.in_channels, self.height, self.width),
                         device=self.device, dtype=dtype)
        with torch.cuda.device(self.device):
            st = torch.cuda.current_stream(self.device).cuda_stream
            _lib.check(L.tsm_net_input_grad(self.h, gx.data_ptr(), _DT[dtype], st))
        return gx

    def dp_init(self, group=None, bucket_bytes=0):
        """Create this rank's NCCL communicator; the unique id travels through
        torch.distributed (plumbing only — the allreduce runs inside the
        library, overlapped with backward)."""
        import torch.distributed as dist
        rank, world = dist.get_rank(group), dist.get_world_size(group)
        buf = (C.c_char * 128)()
        if rank == 0:
            _lib.check(L.tsm_nccl_unique_id(buf))
        obj = [bytes(buf)]
        dist.broadcast_object_list(obj, src=0, group=group)
        C.memmove(buf, obj[0], 128)
        with torch.cuda.device(self.device):
            _lib.check(L.tsm_net_dp_init(self.h, buf, rank, world, bucket_bytes))
        self.world = world
        return self
