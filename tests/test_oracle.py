"""CPU: pin the C restatement (oracle/tsm_oracle.c) against the reference's
golden vectors (tests/golden, generated from the reference built in place)
and, where oracle/_ref is built, against the reference library directly."""
import json

import numpy as np
import pytest

from pathlib import Path

GOLDEN = Path(__file__).resolve().parent / "golden"


def test_kat_shift_and_adjoint(port, golden):
    # kernels_test.cpp:41-55
    k = golden["kat_shift"]
    x = np.array(k["x"]).reshape(k["shape"])
    assert np.array_equal(port.shift(x, tuple(k["fraction"])).ravel(), np.array(k["y"]))
    assert np.array_equal(port.shift(x, tuple(k["fraction"]), adjoint=True).ravel(),
                          np.array(k["adjoint"]))
    y = port.shift(x)
    for t in range(4):
        assert y[0, t, 0, 0, 0] == (0.0 if t == 0 else 100.0 * (t - 1))
        assert y[0, t, 1, 0, 0] == (0.0 if t == 3 else 100.0 * (t + 1) + 1)
        for c in range(2, 8):
            assert y[0, t, c, 0, 0] == 100.0 * t + c


def test_fraction_zero_is_identity(port):
    # kernels_test.cpp:57-61
    x = port.random_normal((2, 5, 4, 3, 3), 11)
    assert np.array_equal(port.shift(x, (0, 1)), x)


def test_validate_matches_reference(port, golden):
    # kernels_test.cpp:63-67 and more
    from oracle.oracle import ValidationError
    for v in golden["validate"]:
        if v["ok"]:
            port.split(v["channels"], (v["num"], v["den"]))
        else:
            with pytest.raises(ValidationError):
                port.split(v["channels"], (v["num"], v["den"]))


def test_seed_sweep_digests(port, golden):
    # kernels_test.cpp:69-84: shapes (1+s%2, 3+s%4, 8, 2, 3), 100 seeds
    for case in golden["seed_sweep"]:
        s, seed, frac = tuple(case["shape"]), case["seed"], tuple(case["fraction"])
        x = port.random_normal(s, seed * 2 + 1)
        y = port.random_normal(s, seed * 2 + 2)
        assert f"{port.fnv1a64(port.shift(x, frac)):016x}" == case["shift_x"]
        assert case["shift_x"] == case["shift_x_serial"]
        assert f"{port.fnv1a64(port.shift(y, frac, adjoint=True)):016x}" == case["adjoint_y"]
        lhs = float(np.dot(port.shift(x, frac).ravel(), y.ravel()))
        rhs = float(np.dot(x.ravel(), port.shift(y, frac, adjoint=True).ravel()))
        assert abs(lhs - rhs) / max(abs(lhs), abs(rhs), 1e-300) < 1e-12


def test_boundary_cells(port, golden):
    # acceptance_test.cpp:124-127
    y = port.shift(np.ones((1, 4, 8, 3, 3)))
    b = golden["boundary"]
    assert y[0, 0, 0, 0, 0] == b["y_0_0_0"] == 0.0
    assert y[0, 3, 1, 0, 0] == b["y_0_3_1"] == 0.0
    assert y[0, 1, 0, 0, 0] == b["y_0_1_0"] == 1.0
    assert y[0, 0, 2, 0, 0] == b["y_0_0_2"] == 1.0
    assert not np.signbit(y).any()  # the fill is +0.0, never -0.0


@pytest.mark.parametrize("seed", ["1", "42"])
def test_c1_digests_fp32(port, golden, seed):
    d = golden["c1"][seed]
    x = port.random_normal((2, 8, 64, 56, 56), int(seed)).astype(np.float32)
    assert f"{port.fnv1a64(x):016x}" == d["x_f32"]
    assert f"{port.fnv1a64(port.shift(x)):016x}" == d["shift_f32"]
    assert f"{port.fnv1a64(port.shift(x, adjoint=True)):016x}" == d["adjoint_f32"]


def test_rng_matches_reference(port, ref):
    for seed, shape in [(1, (2, 3, 4, 5, 6)), (43, (1, 4, 8, 5, 5)), (12345, (1, 1, 1, 1, 1001))]:
        assert np.array_equal(port.random_normal(shape, seed), ref.random_normal(shape, seed))
        assert np.array_equal(port.random_normal(shape, seed, 0.1),
                              ref.random_normal(shape, seed, 0.1))
        assert np.array_equal(port.random_uniform(shape, seed, -2.0, 2.0),
                              ref.random_uniform(shape, seed, -2.0, 2.0))


# kernels_test.cpp:108-119 geometry cases (frame-local and 3-D)
CONV_CASES = [
    ((1, 1, 3, 8, 8), 4, (1, 3, 3), (1, 1, 1), (0, 1, 1)),
    ((2, 1, 2, 9, 7), 3, (1, 3, 3), (1, 2, 2), (0, 1, 1)),
    ((1, 1, 1, 11, 11), 2, (1, 7, 7), (1, 2, 2), (0, 3, 3)),
    ((1, 1, 4, 5, 5), 6, (1, 1, 1), (1, 1, 1), (0, 0, 0)),
    ((1, 6, 3, 6, 6), 4, (3, 3, 3), (1, 1, 1), (1, 1, 1)),
    ((1, 4, 8, 4, 4), 8, (1, 1, 1), (1, 2, 2), (0, 0, 0)),
]


@pytest.mark.parametrize("case", CONV_CASES)
def test_conv_matches_reference_bitwise(port, ref, case):
    shape, cout, k, s, p = case
    x = port.random_normal(shape, 101)
    w = port.random_normal((cout, shape[2]) + k, 102)
    b = port.random_normal((cout,), 103)
    y = port.conv_forward(x, w, b, k, s, p)
    assert np.array_equal(y, ref.conv_forward(x, w, b, k, s, p))
    assert np.array_equal(y, ref.conv_forward(x, w, b, k, s, p, serial=True))
    gy = port.random_normal(y.shape, 104)
    gx, gw, gb = port.conv_backward(x, w, gy, k, s, p)
    rgx, rgw, rgb = ref.conv_backward(x, w, b, gy, k, s, p)
    assert np.array_equal(gx, rgx) and np.array_equal(gw, rgw) and np.array_equal(gb, rgb)


def _block_cases():
    meta = json.loads((GOLDEN / "block_golden.json").read_text())
    return meta


@pytest.mark.parametrize("case", _block_cases(), ids=lambda c: c["name"])
def test_block_port_matches_golden(port, case):
    z = np.load(GOLDEN / "block_golden.npz")
    n = case["name"]
    ws = [z[f"{n}/w{j}"] if f"{n}/w{j}" in z else None for j in range(8)]
    y, gx, gws = port.block(z[f"{n}/x"], ws, case["c_out"], case["stride"], tuple(case["shift"]),
                            gy=z[f"{n}/gy"])
    # Same fp64 operations in the same order as the reference: bit-exact.
    assert np.array_equal(y, z[f"{n}/y"])
    assert np.array_equal(gx, z[f"{n}/gx"])
    for j in range(8):
        if ws[j] is not None:
            assert np.array_equal(gws[j], z[f"{n}/gw{j}"]), j


def test_gradcheck_micro_tsm_reference(ref):
    # gradcheck_test.cpp:8-14 — pins the reference build itself.
    x = ref.random_normal((1, 4, 8, 5, 5), 43)
    err, n = ref.gradcheck("micro-tsm", x, 1e-5, 42)
    assert n == 772 + x.size
    assert err < 1e-5
