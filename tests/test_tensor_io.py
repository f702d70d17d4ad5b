"""The reference's binary tensor fixture format (tensor.cpp:78-110) and the
GPU-backed shift-demo CLI (vidperf.cpp:299-336; cli_test.cpp:176-198).

CPU: our reader/writer against the reference's own write_tensor/read_tensor
(oracle/_ref) both ways, byte-identical files, the reference's error cases;
the CLI's validation exit code.  GPU: the cli_test round trip."""
import subprocess
import sys

import numpy as np
import pytest

from paper_1910_00932_b200 import ValidationError
from paper_1910_00932_b200.cli import fmt_double
from paper_1910_00932_b200.tensor_io import read_tensor, write_tensor

ROOT = __import__("pathlib").Path(__file__).resolve().parents[1]


def test_round_trip_against_reference(tmp_path, ref):
    x = ref.random_normal((2, 3, 4, 5, 6), 7)
    ours, theirs = tmp_path / "ours.bin", tmp_path / "theirs.bin"
    write_tensor(x, ours)
    ref.write_tensor(x, theirs)
    assert ours.read_bytes() == theirs.read_bytes()        # identical files
    assert np.array_equal(ref.read_tensor(ours), x)        # reference reads ours
    assert np.array_equal(read_tensor(theirs), x)          # we read the reference's
    assert read_tensor(ours).shape == (2, 3, 4, 5, 6)


@pytest.mark.parametrize("case", ["header", "payload", "trailing", "zero", "missing"])
def test_read_errors_match_reference(tmp_path, ref, case):
    path = tmp_path / f"{case}.bin"
    good = np.arange(2 * 1 * 2 * 1 * 3, dtype=np.float64).reshape(2, 1, 2, 1, 3)
    write_tensor(good, path)
    data = path.read_bytes()
    if case == "header":
        path.write_bytes(data[:12])
    elif case == "payload":
        path.write_bytes(data[:-8])
    elif case == "trailing":
        path.write_bytes(data + b"\0")
    elif case == "zero":
        path.write_bytes(np.array([2, 0, 2, 1, 3], dtype="<u4").tobytes())
    else:
        path = tmp_path / "nope.bin"
    with pytest.raises(ValidationError) as ours:
        read_tensor(path)
    with pytest.raises(Exception) as theirs:
        ref.read_tensor(path)
    assert type(theirs.value).__name__ == "ValidationError"
    assert str(ours.value) == str(theirs.value)


def test_fmt_double():
    # fmt "{}" (shortest round trip) as printed by the reference's shift-demo
    assert [fmt_double(v) for v in (0.0, 7.0, 301.0, -0.0, 0.5, 1e16, 1e15, 1.5e-5, 0.1)] == \
        ["0", "7", "301", "-0", "0.5", "1e+16", "1000000000000000", "1.5e-05", "0.1"]


def _cli(*args):
    return subprocess.run([sys.executable, "-m", "paper_1910_00932_b200", *args],
                          capture_output=True, text=True, cwd=ROOT)


def test_cli_rejects_bad_fraction():
    r = _cli("shift-demo", "--channels", "8", "--fraction", "1/3")
    assert r.returncode == 1 and r.stderr.startswith("error: ")


@pytest.mark.gpu
def test_shift_demo_round_trip(tmp_path, ref):
    # cli_test.cpp:176-198 with the reference computing the expectations
    saved, twice = tmp_path / "shift.bin", tmp_path / "shift_twice.bin"
    r = _cli("shift-demo", "--frames", "4", "--channels", "8", "--save", str(saved))
    assert r.returncode == 0, r.stderr
    assert "input (h=0, w=0):" in r.stdout and "shifted (h=0, w=0):" in r.stdout
    x = np.zeros((1, 4, 8, 1, 1))
    for t in range(4):
        for c in range(8):
            x[0, t, c, 0, 0] = 100.0 * t + c
    want = ref.temporal_shift(x, (1, 8))
    assert np.array_equal(read_tensor(saved), want)
    assert np.array_equal(ref.read_tensor(saved), want)
    r2 = _cli("shift-demo", "--in", str(saved), "--save", str(twice))
    assert r2.returncode == 0, r2.stderr
    assert np.array_equal(read_tensor(twice), ref.temporal_shift(want, (1, 8)))
    # the report text, line by line (vidperf.cpp:320-333)
    lines = r.stdout.splitlines()
    assert lines[0] == "temporal shift, fraction 1/8 each way, shape t=4 c=8"
    assert lines[2] == "t0:" + "".join(f" {c:>6}" for c in range(8))
    assert lines[7] == "t0:" + "".join(f" {v:>6}" for v in ["0", "101", "2", "3", "4", "5", "6", "7"])
