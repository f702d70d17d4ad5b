"""ctypes binding of libtsm_b200.so (include/tsm_b200.h).

The product path has no fallback: importing this module raises if the CUDA
library has not been built (`make lib` / ``__graft_entry__.build()``), and
every compute entry point raises if no sm_100 device is present.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

LIB_PATH = Path(__file__).resolve().parent / "libtsm_b200.so"

TSM_OK, TSM_ERR_INVALID, TSM_ERR_ALIAS, TSM_ERR_UNSUPPORTED, TSM_ERR_CUDA, TSM_ERR_NCCL = range(6)
TSM_F32, TSM_BF16, TSM_F64, TSM_F16 = range(4)


class ValidationError(RuntimeError):
    """vidperf::ValidationError (errors.hpp:11-13): bad split, shape or weights."""


class TsmError(RuntimeError):
    """CUDA / NCCL failure (the reference's std::runtime_error class)."""


if not LIB_PATH.exists():
    raise ImportError(
        f"{LIB_PATH} is missing: build the CUDA extension first (`make lib` or "
        "`python -c 'import __graft_entry__ as g; g.build()'`). There is no CPU fallback.")

lib = C.CDLL(str(LIB_PATH))

_i64 = C.c_int64
_vp = C.c_void_p

lib.tsm_last_error.restype = C.c_char_p
lib.tsm_abi_version.restype = C.c_int
lib.tsm_launch_count.restype = C.c_uint64
lib.tsm_validate_shift.argtypes = [_i64] * 5 + [C.POINTER(_i64), C.POINTER(_i64)]
lib.tsm_validate_shift.restype = C.c_int
for _fn in (lib.tsm_shift_fwd, lib.tsm_shift_bwd):
    _fn.argtypes = [_vp, _vp] + [_i64] * 7 + [C.c_int, _vp]
    _fn.restype = C.c_int
lib.tsm_shift_host.argtypes = [_vp, _vp] + [_i64] * 7 + [C.c_int, C.c_int]
lib.tsm_shift_host.restype = C.c_int


_ci = C.c_int
lib.tsm_conv_fwd.argtypes = [_vp] * 5 + [_i64] * 6 + [_ci, _ci, _i64, _i64, _ci, _vp]
lib.tsm_conv_dgrad.argtypes = [_vp] * 6 + [_i64] * 6 + [_ci, _ci, _i64, _i64, _vp]
lib.tsm_conv_wgrad_workspace_bytes.argtypes = [_i64] * 6 + [_ci, _ci]
lib.tsm_conv_wgrad_workspace_bytes.restype = C.c_size_t
lib.tsm_conv_wgrad.argtypes = [_vp] * 5 + [_i64] * 6 + [_ci, _ci, _i64, _i64, _vp]
lib.tsm_weights_to_bf16.argtypes = [_vp] * 3 + [_i64, _i64, _ci, _i64, _vp]
lib.tsm_bias_grad_workspace_bytes.argtypes = [_i64, _i64]
lib.tsm_bias_grad_workspace_bytes.restype = C.c_size_t
lib.tsm_bias_grad.argtypes = [_vp] * 3 + [_i64, _i64, _vp]
lib.tsm_maxpool_fwd.argtypes = [_vp, _vp, _vp] + [_i64] * 4 + [_vp]
lib.tsm_maxpool_bwd.argtypes = [_vp, _vp, _vp] + [_i64] * 4 + [_vp]
lib.tsm_maxpool_fwd.restype = lib.tsm_maxpool_bwd.restype = C.c_int
lib.tsm_layout_to_nthwc.argtypes = [_vp, _ci, _vp] + [_i64] * 5 + [_vp]
lib.tsm_layout_to_ntchw.argtypes = [_vp, _vp, _ci] + [_i64] * 4 + [_vp]
for _fn in (lib.tsm_conv_fwd, lib.tsm_conv_dgrad, lib.tsm_conv_wgrad, lib.tsm_weights_to_bf16,
            lib.tsm_bias_grad, lib.tsm_layout_to_nthwc, lib.tsm_layout_to_ntchw):
    _fn.restype = C.c_int


class BlockDesc(C.Structure):
    _fields_ = [("n", _i64), ("t", _i64), ("h", _i64), ("w", _i64), ("c_in", _i64),
                ("c_out", _i64), ("stride", C.c_int32), ("fold_fwd", _i64), ("fold_bwd", _i64)]


class BlockPtrs(C.Structure):
    _fields_ = [(k, _vp) for k in ("w1", "b1", "w2", "b2", "w3", "b3", "wp", "bp")]


lib.tsm_block_workspace_bytes.argtypes = [C.POINTER(BlockDesc)]
lib.tsm_block_workspace_bytes.restype = C.c_size_t
lib.tsm_block_fwd.argtypes = [C.POINTER(BlockDesc), C.POINTER(BlockPtrs), _vp, _vp, _vp, _vp]
lib.tsm_block_fwd.restype = C.c_int
lib.tsm_block_bwd.argtypes = [C.POINTER(BlockDesc), C.POINTER(BlockPtrs), _vp, _vp, _vp, _vp,
                              C.POINTER(BlockPtrs), _vp, _vp]
lib.tsm_block_bwd.restype = C.c_int


def check(status: int) -> None:
    if status == TSM_OK:
        return
    msg = lib.tsm_last_error().decode(errors="replace")
    if status == TSM_ERR_INVALID:
        raise ValidationError(msg)
    if status == TSM_ERR_ALIAS:
        raise ValueError(msg)
    if status == TSM_ERR_UNSUPPORTED:
        raise NotImplementedError(msg)
    raise TsmError(msg)


def launch_count() -> int:
    return int(lib.tsm_launch_count())


lib.tsm_probe_shift_conv1.argtypes = [_i64, _i64]
lib.tsm_probe_shift_conv1.restype = C.c_int
lib.tsm_probe_shift_conv1_read.argtypes = [C.POINTER(C.c_int), C.POINTER(C.c_double),
                                           C.POINTER(_i64)]
lib.tsm_probe_shift_conv1_read.restype = C.c_int


def probe_shift_conv1(c_in: int, c_out: int = 0) -> None:
    """Start (c_in > 0) or stop (c_in == 0) event timing of the fused shift +
    1x1 conv forward launches with these channels inside the bottleneck units
    (bench.py's in-step roofline)."""
    check(lib.tsm_probe_shift_conv1(c_in, c_out))


def probe_shift_conv1_read():
    """(launches, mean launch µs, pixels per launch) of the recorded launches."""
    n, us, px = C.c_int(), C.c_double(), _i64()
    check(lib.tsm_probe_shift_conv1_read(C.byref(n), C.byref(us), C.byref(px)))
    return n.value, us.value, px.value
