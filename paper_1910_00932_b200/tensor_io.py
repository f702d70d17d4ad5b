"""The reference's binary tensor fixture format (tensor.cpp:78-110), the
oracle-comparison interchange format of SPEC.md:253.

Layout: five little-endian uint32 dims (n, t, c, h, w), then n*t*c*h*w fp64
values in NTCHW order, nothing after.  Reading rejects a zero dimension, a
short header, a short payload and trailing bytes with the reference's
messages (ValidationError).  Host-side IO only — no compute."""
from __future__ import annotations

import os

import numpy as np

from ._lib import ValidationError

_HEADER = np.dtype("<u4")
_PAYLOAD = np.dtype("<f8")


def write_tensor(tensor, path: str | os.PathLike) -> None:
    """write_tensor (tensor.cpp:78-89): any 5-D array-like, stored as fp64."""
    arr = np.ascontiguousarray(np.asarray(tensor, dtype=np.float64))
    if arr.ndim != 5:
        raise ValidationError(f"write_tensor: expected a 5-D tensor, got {arr.ndim}-D")
    try:
        with open(path, "wb") as f:
            f.write(np.asarray(arr.shape, dtype=_HEADER).tobytes())
            f.write(arr.astype(_PAYLOAD, copy=False).tobytes())
    except OSError:
        raise ValidationError(f"cannot write tensor '{path}'") from None


def read_tensor(path: str | os.PathLike) -> np.ndarray:
    """read_tensor (tensor.cpp:91-110) -> float64 array [n][t][c][h][w]."""
    try:
        with open(path, "rb") as f:
            data = f.read()
    except OSError:
        raise ValidationError(f"cannot open tensor '{path}'") from None
    if len(data) < 20:
        raise ValidationError(f"tensor '{path}' truncated in header")
    dims = tuple(int(d) for d in np.frombuffer(data[:20], dtype=_HEADER))
    if any(d == 0 for d in dims):
        raise ValidationError(f"tensor '{path}' has a zero dimension")
    count = int(np.prod(dims, dtype=np.int64))
    need = 20 + 8 * count
    if len(data) < need:
        raise ValidationError(f"tensor '{path}' truncated in payload")
    if len(data) > need:
        raise ValidationError(f"tensor '{path}' has trailing bytes")
    return np.frombuffer(data[20:need], dtype=_PAYLOAD).reshape(dims).astype(np.float64)
