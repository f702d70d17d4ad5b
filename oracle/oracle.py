"""TEST INFRASTRUCTURE ONLY — ctypes views of the two CPU oracles.

* ``Port``: oracle/libtsm_oracle.so, the plain-C restatement (tsm_oracle.c).
* ``Reference``: oracle/_ref/libvidperf_ref.so, the unmodified reference
  library compiled in place from /root/reference (oracle/Makefile) plus a C
  shim (ref_capi.cpp).

Only tests/, ``__graft_entry__.smoke()`` and bench.py's CPU-baseline legs may
import this module.  The product package (paper_1910_00932_b200) never does.
All tensors are numpy arrays in the reference layout [N][T][C][H][W].
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
PORT_SO = HERE / "libtsm_oracle.so"
REF_SO = HERE / "_ref" / "libvidperf_ref.so"

_dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_i64p = C.POINTER(C.c_int64)


class ValidationError(RuntimeError):
    """Mirror of vidperf::ValidationError (errors.hpp:11-13)."""


def _shape(s):
    return (C.c_int64 * 5)(*[int(v) for v in s])


def _ints(v):
    return (C.c_int * 3)(*[int(a) for a in v])


def _ptr(a):
    return a.ctypes.data_as(C.c_void_p) if a is not None else None


def _wvec(ws):
    arr = (C.c_void_p * 8)()
    for i, w in enumerate(ws):
        arr[i] = _ptr(w) if w is not None else None
    return arr


class Port:
    """The C restatement.  Loaded lazily; raises if not built."""

    def __init__(self, path: Path = PORT_SO):
        if not path.exists():
            raise FileNotFoundError(f"{path} missing: run `make -C oracle`")
        self.lib = L = C.CDLL(str(path))
        L.tso_random_normal.argtypes = [C.c_int64, C.c_uint64, C.c_double, C.c_void_p]
        L.tso_random_uniform.argtypes = [C.c_int64, C.c_uint64, C.c_double, C.c_double, C.c_void_p]
        L.tso_fnv1a64.argtypes = [C.c_void_p, C.c_size_t]
        L.tso_fnv1a64.restype = C.c_uint64
        L.tso_validate_shift.argtypes = [C.c_int64] * 5 + [_i64p, _i64p]
        L.tso_shift_bytes.argtypes = [C.c_void_p, C.c_void_p] + [C.c_int64] * 7 + [C.c_int]
        L.tso_conv_forward.argtypes = [C.c_void_p, _i64p, C.c_int64, C.c_void_p, C.c_void_p,
                                       C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, _i64p]
        L.tso_conv_backward.argtypes = [C.c_void_p, _i64p, C.c_int64, C.c_void_p, C.c_void_p,
                                        C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                        C.c_void_p, C.c_void_p]
        L.tso_block.argtypes = [C.c_void_p, _i64p, C.c_int64, C.c_int, C.c_int64, C.c_int64,
                                C.c_void_p, C.c_void_p, _i64p, C.c_void_p, C.c_void_p, C.c_void_p]
        L.tso_block.restype = C.c_int
        L.tso_block_ex.argtypes = L.tso_block.argtypes + [C.c_int]
        L.tso_block_ex.restype = C.c_int

    # tensor.cpp:41-47
    def random_normal(self, shape, seed, stddev=1.0):
        out = np.empty(int(np.prod(shape)), np.float64)
        self.lib.tso_random_normal(out.size, seed, stddev, _ptr(out))
        return out.reshape(shape)

    def random_uniform(self, shape, seed, lo, hi):
        out = np.empty(int(np.prod(shape)), np.float64)
        self.lib.tso_random_uniform(out.size, seed, lo, hi, _ptr(out))
        return out.reshape(shape)

    def fnv1a64(self, arr) -> int:
        a = np.ascontiguousarray(arr)
        return int(self.lib.tso_fnv1a64(_ptr(a), a.nbytes))

    def split(self, channels, fwd=(1, 8), bwd=None):
        bwd = fwd if bwd is None else bwd
        f, b = C.c_int64(), C.c_int64()
        if self.lib.tso_validate_shift(fwd[0], fwd[1], bwd[0], bwd[1], channels,
                                       C.byref(f), C.byref(b)):
            raise ValidationError(f"shift {fwd}/{bwd} does not split {channels} channels")
        return f.value, b.value

    def shift(self, x, fraction=(1, 8), adjoint=False, bwd_fraction=None):
        """kernels.cpp:97-157 on any dtype (bitwise copy)."""
        x = np.ascontiguousarray(x)
        n, t, c, h, w = x.shape
        f, b = self.split(c, fraction, bwd_fraction)
        out = np.empty_like(x)
        self.lib.tso_shift_bytes(_ptr(x), _ptr(out), n, t, c, h * w, f, b, x.itemsize,
                                 int(adjoint))
        return out

    def conv_forward(self, x, w, b, kernel, stride=(1, 1, 1), padding=(0, 0, 0)):
        x = np.ascontiguousarray(x, np.float64)
        ys = (C.c_int64 * 5)()
        cout = w.shape[0]
        args = (_ptr(x), _shape(x.shape), cout, _ints(kernel), _ints(stride), _ints(padding),
                _ptr(np.ascontiguousarray(w, np.float64)), _ptr(np.ascontiguousarray(b, np.float64)))
        self.lib.tso_conv_forward(*args, None, ys)
        y = np.empty(tuple(ys), np.float64)
        self.lib.tso_conv_forward(*args, _ptr(y), ys)
        return y

    def conv_backward(self, x, w, gy, kernel, stride=(1, 1, 1), padding=(0, 0, 0)):
        x = np.ascontiguousarray(x, np.float64)
        w = np.ascontiguousarray(w, np.float64)
        gy = np.ascontiguousarray(gy, np.float64)
        gx = np.empty_like(x)
        gw = np.empty_like(w)
        gb = np.empty(w.shape[0], np.float64)
        self.lib.tso_conv_backward(_ptr(x), _shape(x.shape), w.shape[0], _ints(kernel),
                                   _ints(stride), _ints(padding), _ptr(w), _ptr(gy), _ptr(gx),
                                   _ptr(gw), _ptr(gb))
        return gx, gw, gb

    def block(self, x, weights, c_out, stride=1, shift=(1, 8), gy=None, bf16_storage=False):
        """Bottleneck unit fwd (+bwd if gy).  weights = [w1,b1,w2,b2,w3,b3,wp,bp].
        bf16_storage=True rounds stored activations/gradients to bf16 like the
        GPU path (test-only sharpening; False is the reference algorithm)."""
        if bf16_storage:
            fn = lambda *a: self.lib.tso_block_ex(*a, 1)  # noqa: E731
        else:
            fn = self.lib.tso_block
        return _block(fn, x, weights, c_out, stride, shift, gy)


def _block(fn, x, weights, c_out, stride, shift, gy):
    x = np.ascontiguousarray(x, np.float64)
    ws = [None if w is None else np.ascontiguousarray(w, np.float64) for w in weights]
    ys = (C.c_int64 * 5)()
    n, t, cin, h, w_ = x.shape
    ho = (h + 2 - 3) // stride + 1
    wo = (w_ + 2 - 3) // stride + 1
    y = np.empty((n, t, c_out, ho, wo), np.float64)
    gx = gws = None
    if gy is not None:
        gy = np.ascontiguousarray(gy, np.float64)
        gx = np.empty_like(x)
        gws = [None if w is None else np.empty_like(w) for w in ws]
    rc = fn(_ptr(x), _shape(x.shape), c_out, stride, shift[0], shift[1], _wvec(ws), _ptr(y), ys,
            _ptr(gy), _ptr(gx), _wvec(gws) if gws else None)
    if rc:
        raise ValidationError("bad block configuration")
    assert tuple(ys) == y.shape, (tuple(ys), y.shape)
    return (y, gx, gws) if gy is not None else y


class Reference:
    """The unmodified reference library (vidperf), via oracle/_ref."""

    def __init__(self, path: Path = REF_SO, mode: int = C.DEFAULT_MODE):
        if not path.exists():
            raise FileNotFoundError(f"{path} missing: run `make -C oracle ref` where "
                                    "/root/reference exists")
        self.lib = L = C.CDLL(str(path), mode=mode)
        L.vref_last_error.restype = C.c_char_p
        L.vref_random_normal.argtypes = [_i64p, C.c_uint64, C.c_double, C.c_void_p]
        L.vref_random_uniform.argtypes = [_i64p, C.c_uint64, C.c_double, C.c_double, C.c_void_p]
        L.vref_validate_shift.argtypes = [C.c_int64] * 5
        L.vref_temporal_shift.argtypes = [C.c_void_p, _i64p] + [C.c_int64] * 4 + [C.c_int,
                                                                                 C.c_void_p]
        L.vref_temporal_shift_adjoint.argtypes = [C.c_void_p, _i64p] + [C.c_int64] * 4 + [
            C.c_void_p]
        L.vref_time_shift.argtypes = [_i64p, C.c_uint64, C.c_int64, C.c_int, C.c_int, C.c_int]
        L.vref_time_shift.restype = C.c_double
        L.vref_conv_forward.argtypes = [C.c_void_p, _i64p, C.c_int64, C.c_void_p, C.c_void_p,
                                        C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_void_p,
                                        _i64p]
        L.vref_conv_backward.argtypes = [C.c_void_p, _i64p, C.c_int64, C.c_void_p, C.c_void_p,
                                         C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                         C.c_void_p, C.c_void_p, C.c_void_p]
        L.vref_max_pool.argtypes = [C.c_void_p, _i64p, C.c_void_p, C.c_void_p, C.c_void_p,
                                    C.c_void_p, C.c_void_p, C.c_void_p, _i64p]
        L.vref_block.argtypes = [C.c_void_p, _i64p, C.c_int64, C.c_int, C.c_int64, C.c_int64,
                                 C.c_void_p, C.c_void_p, _i64p, C.c_void_p, C.c_void_p,
                                 C.c_void_p]
        L.vref_net_create.argtypes = [C.c_char_p, C.c_int64, C.c_int64, C.c_uint64]
        L.vref_net_create.restype = C.c_void_p
        L.vref_net_create_sized.argtypes = [C.c_int64, C.c_int64, C.c_uint64]
        L.vref_net_create_sized.restype = C.c_void_p
        L.vref_time_loss_gradients.argtypes = [C.c_void_p, C.c_int64, C.c_int]
        L.vref_time_loss_gradients.restype = C.c_double
        L.vref_net_destroy.argtypes = [C.c_void_p]
        L.vref_net_param_count.argtypes = [C.c_void_p]
        L.vref_net_param_count.restype = C.c_int64
        L.vref_net_get_params.argtypes = [C.c_void_p, C.c_void_p]
        L.vref_net_set_params.argtypes = [C.c_void_p, C.c_void_p]
        L.vref_net_forward.argtypes = [C.c_void_p, C.c_void_p, _i64p, C.c_void_p, _i64p]
        L.vref_net_loss_gradients.argtypes = [C.c_void_p, C.c_void_p, _i64p, C.c_void_p,
                                              C.c_void_p, C.c_void_p]
        L.vref_gradcheck.argtypes = [C.c_char_p, C.c_int64, C.c_int64, C.c_void_p, _i64p,
                                     C.c_double, C.c_uint64, C.c_void_p, C.c_void_p]
        L.vref_write_tensor.argtypes = [C.c_void_p, _i64p, C.c_char_p]
        L.vref_step_time.argtypes = [C.c_void_p, C.c_int64, C.c_int64, C.c_int64, C.c_int,
                                     C.c_double, C.c_int, C.c_void_p]
        L.vref_observed_scalability.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_void_p]
        L.vref_read_tensor.argtypes = [C.c_char_p, _i64p, C.c_void_p]

    def _check(self, rc):
        if rc == 1:
            raise ValidationError(self.lib.vref_last_error().decode())
        if rc:
            raise RuntimeError(self.lib.vref_last_error().decode())

    def random_normal(self, shape, seed, stddev=1.0):
        out = np.empty(shape, np.float64)
        self._check(self.lib.vref_random_normal(_shape(shape), seed, stddev, _ptr(out)))
        return out

    def random_uniform(self, shape, seed, lo, hi):
        out = np.empty(shape, np.float64)
        self._check(self.lib.vref_random_uniform(_shape(shape), seed, lo, hi, _ptr(out)))
        return out

    def step_time(self, prof, flops, params, input_bytes, per_gpu_batch, flop_mult=3.0,
                  ring=True):
        """vidperf::step_time (sim.cpp:132-144) -> (t_compute, t_io, t_comm, t_step)."""
        pr = np.asarray(prof, dtype=np.float64)
        out = np.zeros(4)
        self._check(self.lib.vref_step_time(_ptr(pr), flops, params, input_bytes, per_gpu_batch,
                                            flop_mult, int(ring), _ptr(out)))
        return tuple(out)

    def observed_scalability(self, timings):
        """vidperf::observed_scalability (sim.cpp:195-215)."""
        nodes = np.asarray([t[0] for t in timings], dtype=np.int64)
        secs = np.asarray([t[1] for t in timings], dtype=np.float64)
        out = np.zeros(len(timings))
        self._check(self.lib.vref_observed_scalability(_ptr(nodes), _ptr(secs), len(timings),
                                                       _ptr(out)))
        return list(zip(nodes.tolist(), out.tolist()))

    def write_tensor(self, x, path):
        """vidperf::write_tensor (tensor.cpp:78-89)."""
        x = np.ascontiguousarray(x, dtype=np.float64)
        self._check(self.lib.vref_write_tensor(_ptr(x), _shape(x.shape), str(path).encode()))

    def read_tensor(self, path):
        """vidperf::read_tensor (tensor.cpp:91-110)."""
        shape = (C.c_int64 * 5)()
        self._check(self.lib.vref_read_tensor(str(path).encode(), shape, None))
        out = np.empty(tuple(shape), dtype=np.float64)
        self._check(self.lib.vref_read_tensor(str(path).encode(), shape, _ptr(out)))
        return out

    def validate_shift(self, channels, fwd=(1, 8), bwd=None):
        bwd = fwd if bwd is None else bwd
        self._check(self.lib.vref_validate_shift(fwd[0], fwd[1], bwd[0], bwd[1], channels))

    def temporal_shift(self, x, fraction=(1, 8), serial=False, bwd_fraction=None):
        bwd = fraction if bwd_fraction is None else bwd_fraction
        x = np.ascontiguousarray(x, np.float64)
        out = np.empty_like(x)
        self._check(self.lib.vref_temporal_shift(_ptr(x), _shape(x.shape), fraction[0],
                                                 fraction[1], bwd[0], bwd[1], int(serial),
                                                 _ptr(out)))
        return out

    def temporal_shift_adjoint(self, y, fraction=(1, 8), bwd_fraction=None):
        bwd = fraction if bwd_fraction is None else bwd_fraction
        y = np.ascontiguousarray(y, np.float64)
        out = np.empty_like(y)
        self._check(self.lib.vref_temporal_shift_adjoint(_ptr(y), _shape(y.shape), fraction[0],
                                                         fraction[1], bwd[0], bwd[1], _ptr(out)))
        return out

    def time_shift(self, shape, seed=1, fold_div=8, adjoint=False, serial=False, iters=5):
        return self.lib.vref_time_shift(_shape(shape), seed, fold_div, int(adjoint), int(serial),
                                        iters)

    def conv_forward(self, x, w, b, kernel, stride=(1, 1, 1), padding=(0, 0, 0), serial=False):
        x = np.ascontiguousarray(x, np.float64)
        ys = (C.c_int64 * 5)()
        args = (_ptr(x), _shape(x.shape), w.shape[0], _ints(kernel), _ints(stride),
                _ints(padding), _ptr(np.ascontiguousarray(w, np.float64)),
                _ptr(np.ascontiguousarray(b, np.float64)), int(serial))
        self._check(self.lib.vref_conv_forward(*args, None, ys))
        y = np.empty(tuple(ys), np.float64)
        self._check(self.lib.vref_conv_forward(*args, _ptr(y), ys))
        return y

    def conv_backward(self, x, w, b, gy, kernel, stride=(1, 1, 1), padding=(0, 0, 0)):
        x = np.ascontiguousarray(x, np.float64)
        w = np.ascontiguousarray(w, np.float64)
        b = np.ascontiguousarray(b, np.float64)
        gy = np.ascontiguousarray(gy, np.float64)
        gx, gw, gb = np.empty_like(x), np.empty_like(w), np.empty_like(b)
        self._check(self.lib.vref_conv_backward(_ptr(x), _shape(x.shape), w.shape[0],
                                                _ints(kernel), _ints(stride), _ints(padding),
                                                _ptr(w), _ptr(b), _ptr(gy), _ptr(gx), _ptr(gw),
                                                _ptr(gb)))
        return gx, gw, gb

    def max_pool(self, x, kernel, stride, padding, gy=None):
        x = np.ascontiguousarray(x, np.float64)
        ys = (C.c_int64 * 5)()
        self._check(self.lib.vref_max_pool(_ptr(x), _shape(x.shape), _ints(kernel),
                                           _ints(stride), _ints(padding), None, None, None, ys))
        y = np.empty(tuple(ys), np.float64)
        gx = np.empty_like(x) if gy is not None else None
        gy = None if gy is None else np.ascontiguousarray(gy, np.float64)
        self._check(self.lib.vref_max_pool(_ptr(x), _shape(x.shape), _ints(kernel),
                                           _ints(stride), _ints(padding), _ptr(gy), _ptr(y),
                                           _ptr(gx), ys))
        return (y, gx) if gy is not None else y

    def block(self, x, weights, c_out, stride=1, shift=(1, 8), gy=None):
        return _block(self.lib.vref_block, x, weights, c_out, stride, shift, gy)

    # ---- Network (net.hpp:15-54) -------------------------------------------
    def net(self, preset="micro-tsm", shift=(1, 8), seed=42):
        return RefNetwork(self, preset, shift, seed)

    def net_sized(self, h, w, seed=42):
        """vidperf::Network(build_tsm8f() with input extent h x w, seed)
        (ref_capi.cpp vref_net_create_sized; init order unchanged)."""
        return RefNetwork(self, None, None, seed, hw=(h, w))

    def time_train_clip(self, h=64, w=64, clips=1, iters=1, seed=42):
        """Seconds per Network::loss_gradients over `clips` clips of
        build_tsm8f() with the input spatial extent set to h x w."""
        hdl = self.lib.vref_net_create_sized(h, w, seed)
        if not hdl:
            raise ValidationError(self.lib.vref_last_error().decode())
        try:
            return self.lib.vref_time_loss_gradients(hdl, clips, iters)
        finally:
            self.lib.vref_net_destroy(hdl)

    def gradcheck(self, preset, x, eps, seed, shift=(1, 8)):
        x = np.ascontiguousarray(x, np.float64)
        mr, n = C.c_double(), C.c_int64()
        self._check(self.lib.vref_gradcheck(preset.encode(), shift[0], shift[1], _ptr(x),
                                            _shape(x.shape), eps, seed, C.byref(mr), C.byref(n)))
        return mr.value, n.value


class RefNetwork:
    def __init__(self, ref: Reference, preset, shift, seed, hw=None):
        self.ref = ref
        if hw is not None:
            self.h = ref.lib.vref_net_create_sized(hw[0], hw[1], seed)
        else:
            self.h = ref.lib.vref_net_create(preset.encode(), shift[0], shift[1], seed)
        if not self.h:
            raise ValidationError(ref.lib.vref_last_error().decode())

    def __del__(self):
        if getattr(self, "h", None):
            self.ref.lib.vref_net_destroy(self.h)
            self.h = None

    def param_count(self):
        return self.ref.lib.vref_net_param_count(self.h)

    def param_vector(self):
        out = np.empty(self.param_count(), np.float64)
        self.ref.lib.vref_net_get_params(self.h, _ptr(out))
        return out

    def set_params(self, v):
        v = np.ascontiguousarray(v, np.float64)
        assert v.size == self.param_count()
        self.ref.lib.vref_net_set_params(self.h, _ptr(v))

    def forward(self, x):
        x = np.ascontiguousarray(x, np.float64)
        ys = (C.c_int64 * 5)()
        self.ref._check(self.ref.lib.vref_net_forward(self.h, _ptr(x), _shape(x.shape), None, ys))
        y = np.empty(tuple(ys), np.float64)
        self.ref._check(self.ref.lib.vref_net_forward(self.h, _ptr(x), _shape(x.shape), _ptr(y),
                                                      ys))
        return y

    def loss_gradients(self, x):
        x = np.ascontiguousarray(x, np.float64)
        loss = C.c_double()
        gp = np.empty(self.param_count(), np.float64)
        gx = np.empty_like(x)
        self.ref._check(self.ref.lib.vref_net_loss_gradients(self.h, _ptr(x), _shape(x.shape),
                                                             C.byref(loss), _ptr(gp), _ptr(gx)))
        return loss.value, gp, gx


def available_reference() -> bool:
    return REF_SO.exists()


def threads() -> int:
    return int(os.environ.get("OMP_NUM_THREADS", os.cpu_count() or 1))
