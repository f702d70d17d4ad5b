"""GPU-backed ``shift-demo`` (vidperf.cpp:299-336, options :431-439).

    python -m paper_1910_00932_b200 shift-demo [--frames 4] [--channels 8]
        [--height 1] [--width 1] [--fraction 1/8] [--in PATH] [--save PATH]
        [--out PATH]

Same input (a fixture from --in, else the structured grid value = 100t + c),
same report text, same fixture output; the shift itself runs on the GPU
through the C ABI (``tsm_shift_host``: host fp64 in, H2D, sm_100a kernel,
D2H).  Exit codes follow vidperf.cpp:476-484: ValidationError -> 1
("error: ..."), anything else -> 2 ("internal error: ...")."""
from __future__ import annotations

import argparse
import sys

import numpy as np

from ._lib import ValidationError
from .shift import ShiftConfig, parse_rational, temporal_shift_host, validate_shift
from .tensor_io import read_tensor, write_tensor


def fmt_double(v: float) -> str:
    """fmt's shortest round-trip formatting of a double ("{}"): Python's repr
    uses the same digits and the same fixed/scientific switch (exponent < -4
    or >= 16); fmt drops the ".0" of integral values."""
    s = repr(float(v))
    return s[:-2] if s.endswith(".0") else s


def emit(text: str, out_path: str) -> None:
    """emit (vidperf.cpp:23-31)."""
    if not out_path:
        sys.stdout.write(text)
        return
    try:
        with open(out_path, "wb") as f:
            f.write(text.encode())
    except OSError:
        raise ValidationError(f"cannot write '{out_path}'") from None


def run_shift_demo(a: argparse.Namespace) -> int:
    if a.in_path:
        x = read_tensor(a.in_path)
    else:
        for name, v in (("frames", a.frames), ("channels", a.channels), ("height", a.height),
                        ("width", a.width)):
            if v <= 0:  # Tensor5D's positive-shape check (tensor.cpp:16-22)
                raise ValidationError(f"shift-demo: {name} must be positive")
        x = np.zeros((1, a.frames, a.channels, a.height, a.width), dtype=np.float64)
        x += (100.0 * np.arange(a.frames)[:, None] + np.arange(a.channels)[None, :])[None, :, :, None, None]
    cfg = ShiftConfig.symmetric(parse_rational(a.fraction))
    validate_shift(cfg, x.shape[2])
    y = temporal_shift_host(np.ascontiguousarray(x), cfg)
    if a.save:
        write_tensor(y, a.save)
    t, c = x.shape[1], x.shape[2]
    text = f"temporal shift, fraction {cfg.fraction_fwd} each way, shape t={t} c={c}\n"

    def grid(v, title):
        g = f"{title} (h=0, w=0):\n"
        for ti in range(t):
            g += f"t{ti}:" + "".join(f" {fmt_double(v[0, ti, ci, 0, 0]):>6}" for ci in range(c)) + "\n"
        return g

    text += grid(x, "input")
    text += grid(y, "shifted")
    emit(text, a.out)
    return 0


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="paper_1910_00932_b200")
    sub = ap.add_subparsers(dest="cmd", required=True)
    sd = sub.add_parser("shift-demo", help="show the temporal shift on a grid (GPU)")
    sd.add_argument("--frames", type=int, default=4)
    sd.add_argument("--channels", type=int, default=8)
    sd.add_argument("--height", type=int, default=1)
    sd.add_argument("--width", type=int, default=1)
    sd.add_argument("--fraction", default="1/8")
    sd.add_argument("--in", dest="in_path", default="")
    sd.add_argument("--save", default="")
    sd.add_argument("--out", default="")
    a = ap.parse_args(argv)
    try:
        return run_shift_demo(a)
    except ValidationError as e:
        print(f"error: {e}", file=sys.stderr)
        return 1
    except Exception as e:  # noqa: BLE001 - the reference's catch-all exit code
        print(f"internal error: {e}", file=sys.stderr)
        return 2


if __name__ == "__main__":
    sys.exit(main())
