"""GPU parity: the sm_100a shift / adjoint against the oracle, bit-exact.

Inputs come from the reference RNG (oracle port, pinned to the reference);
outputs are compared byte-for-byte with the oracle and with the digests of the
reference's own outputs in tests/golden/shift_golden.json."""
import numpy as np
import pytest
import torch

import paper_1910_00932_b200 as tsm

pytestmark = pytest.mark.gpu

F18 = tsm.ShiftConfig.fold_div(8)


def frac_cfg(fr):
    return tsm.ShiftConfig.symmetric(tsm.Rational(*fr))


def to_dev(a, dtype, dev):
    t = torch.from_numpy(np.ascontiguousarray(a))
    return t.to(dev).to(dtype)


def test_kat(golden, cuda):
    k = golden["kat_shift"]
    x = torch.tensor(k["x"], dtype=torch.float64).reshape(k["shape"]).to(cuda)
    y = tsm.temporal_shift(x, frac_cfg(k["fraction"]))
    a = tsm.temporal_shift_adjoint(x, frac_cfg(k["fraction"]))
    assert torch.equal(y.cpu().flatten(), torch.tensor(k["y"], dtype=torch.float64))
    assert torch.equal(a.cpu().flatten(), torch.tensor(k["adjoint"], dtype=torch.float64))


def test_seed_sweep_bit_exact_fp64(port, golden, cuda):
    # kernels_test.cpp:69-84 — digests of the reference's own outputs.
    for case in golden["seed_sweep"]:
        s, seed, fr = tuple(case["shape"]), case["seed"], tuple(case["fraction"])
        x = port.random_normal(s, seed * 2 + 1)
        y = port.random_normal(s, seed * 2 + 2)
        gx = tsm.temporal_shift(to_dev(x, torch.float64, cuda), frac_cfg(fr)).cpu().numpy()
        gy = tsm.temporal_shift_adjoint(to_dev(y, torch.float64, cuda), frac_cfg(fr)).cpu().numpy()
        assert f"{port.fnv1a64(gx):016x}" == case["shift_x"], seed
        assert f"{port.fnv1a64(gy):016x}" == case["adjoint_y"], seed


@pytest.mark.parametrize("seed", ["1", "42"])
def test_c1_fp32_digests(port, golden, cuda, seed):
    d = golden["c1"][seed]
    x = port.random_normal((2, 8, 64, 56, 56), int(seed)).astype(np.float32)
    assert f"{port.fnv1a64(x):016x}" == d["x_f32"]
    xd = to_dev(x, torch.float32, cuda)
    y = tsm.temporal_shift(xd, F18).cpu().numpy()
    a = tsm.temporal_shift_adjoint(xd, F18).cpu().numpy()
    assert f"{port.fnv1a64(y):016x}" == d["shift_f32"]
    assert f"{port.fnv1a64(a):016x}" == d["adjoint_f32"]


SHAPES = [
    # (N,T,C,H,W), fraction — aligned, unaligned (7x7 planes, odd channel counts), tiny
    ((2, 8, 64, 56, 56), (1, 8)),
    ((1, 8, 256, 56, 56), (1, 8)),
    ((2, 8, 2048, 7, 7), (1, 8)),
    ((1, 16, 128, 28, 28), (1, 8)),
    ((3, 5, 9, 7, 5), (1, 3)),
    ((1, 3, 8, 2, 3), (1, 4)),
    ((2, 1, 16, 3, 3), (1, 8)),    # T = 1: both shifted groups are all-zero
    ((1, 4, 8, 1, 1), (1, 2)),     # F + B = C
    ((1, 2, 24, 1, 1), (0, 1)),    # identity
]


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16, torch.float64, torch.float16])
@pytest.mark.parametrize("shape,fr", SHAPES)
def test_shapes_dtypes_bit_exact(port, cuda, shape, fr, dtype):
    x = port.random_normal(shape, 7)
    xd = to_dev(x, dtype, cuda)
    host = xd.cpu()
    raw = host.view(torch.int16) if dtype.itemsize == 2 else host
    xb = raw.numpy()
    for adjoint in (False, True):
        fn = tsm.temporal_shift_adjoint if adjoint else tsm.temporal_shift
        got = fn(xd, frac_cfg(fr)).cpu()
        got = (got.view(torch.int16) if dtype.itemsize == 2 else got).numpy()
        want = port.shift(xb, fr, adjoint=adjoint)
        assert got.tobytes() == want.tobytes(), (shape, fr, dtype, adjoint)


def test_unaligned_pointer_offsets(port, cuda):
    # Views at odd element offsets exercise the element-granular path.
    base = torch.from_numpy(port.random_normal((1, 1, 1, 1, 4 * 8 * 5 * 5 + 1), 3)).float().to(cuda)
    x = base.flatten()[1:].reshape(1, 4, 8, 5, 5)
    out = torch.empty(4 * 8 * 5 * 5 + 1, device=cuda)[1:].reshape(1, 4, 8, 5, 5)
    tsm.temporal_shift(x, F18, out=out)
    assert out.cpu().numpy().tobytes() == port.shift(x.cpu().numpy()).tobytes()


def test_special_values_preserved(cuda):
    x = torch.zeros(1, 3, 8, 2, 2, device=cuda)
    x[:, :, :] = -0.0
    x[0, 1, 0, 0, 0] = float("nan")
    x[0, 1, 3, 1, 1] = float("inf")
    y = tsm.temporal_shift(x, F18)
    # channel 0 at t=0 reads t=-1: literal +0.0, never -0.0
    assert not torch.signbit(y[0, 0, 0]).any()
    assert not torch.signbit(y[0, 2, 1]).any()
    # pass-through keeps -0.0 and the NaN moves with its channel
    assert torch.signbit(y[0, 1, 3, 0, 0])
    assert torch.isnan(y[0, 2, 0, 0, 0])
    assert torch.isinf(y[0, 1, 3, 1, 1])


def test_adjoint_pairing(port, cuda):
    # acceptance_test.cpp:142-153: <shift(u), v> == <u, shift_adj(v)>
    worst = 0.0
    for seed in range(120):
        s = (1, 3 + seed % 5, 8, 2, 2)
        u = to_dev(port.random_normal(s, 1000 + seed * 2), torch.float64, cuda)
        v = to_dev(port.random_normal(s, 1001 + seed * 2), torch.float64, cuda)
        lhs = float((tsm.temporal_shift(u, F18) * v).sum())
        rhs = float((u * tsm.temporal_shift_adjoint(v, F18)).sum())
        worst = max(worst, abs(lhs - rhs) / max(abs(lhs), abs(rhs), 1e-300))
    assert worst < 1e-12


def test_linearity(port, cuda):
    # kernels_test.cpp:86-100
    a = to_dev(port.random_normal((1, 4, 8, 3, 3), 3), torch.float64, cuda)
    b = to_dev(port.random_normal((1, 4, 8, 3, 3), 4), torch.float64, cuda)
    assert torch.equal(tsm.temporal_shift(2 * a + b, F18),
                       2 * tsm.temporal_shift(a, F18) + tsm.temporal_shift(b, F18))


@pytest.mark.parametrize("shape", [(8, 16, 2048, 56, 56), (64, 8, 256, 56, 56)])
def test_full_size_structure(cuda, shape):
    # Largest sweep shapes (C5, bf16, 1.6 GB / 0.8 GB): size-independent checks
    # of the three runs and the +0.0 boundary against plain slicing.
    torch.manual_seed(0)
    x = torch.randn(shape, device=cuda, dtype=torch.bfloat16)
    c = shape[2]
    f = c // 8
    for adjoint in (False, True):
        y = (tsm.temporal_shift_adjoint if adjoint else tsm.temporal_shift)(x, F18)
        lo, hi = (slice(1, None), slice(None, -1))
        g0_dst, g0_src = (hi, lo) if adjoint else (lo, hi)
        assert torch.equal(y[:, g0_dst, :f], x[:, g0_src, :f])
        assert torch.equal(y[:, g0_src, f:2 * f], x[:, g0_dst, f:2 * f])
        assert torch.equal(y[:, :, 2 * f:], x[:, :, 2 * f:])
        edge0 = y[:, -1 if adjoint else 0, :f]
        edge1 = y[:, 0 if adjoint else -1, f:2 * f]
        assert (edge0.view(torch.int16) == 0).all() and (edge1.view(torch.int16) == 0).all()
        del y
    torch.cuda.synchronize()


def test_host_buffer_path_matches_reference(port, cuda):
    x = port.random_normal((2, 8, 64, 56, 56), 1)
    for adjoint in (False, True):
        y = tsm.temporal_shift_host(x, F18, adjoint=adjoint)
        assert y.tobytes() == port.shift(x, adjoint=adjoint).tobytes()


def test_validation_errors_before_launch(cuda):
    x = torch.zeros(1, 2, 12, 2, 2, device=cuda)
    with pytest.raises(tsm.ValidationError):
        tsm.temporal_shift(x, tsm.ShiftConfig.symmetric(tsm.Rational(1, 8)))
    with pytest.raises(tsm.ValidationError):
        tsm.temporal_shift(x, tsm.ShiftConfig(tsm.Rational(1, 2), tsm.Rational(2, 3)))
    with pytest.raises(ValueError):
        _alias(x)


def _alias(x):
    from paper_1910_00932_b200 import _lib
    _lib.check(_lib.lib.tsm_shift_fwd(x.data_ptr(), x.data_ptr() + 16, 1, 2, 8, 2, 2, 1, 1,
                                      _lib.TSM_F32, None))


def test_determinism(port, cuda):
    x = to_dev(port.random_normal((4, 8, 128, 28, 28), 5), torch.bfloat16, cuda)
    ys = [tsm.temporal_shift(x, F18) for _ in range(3)]
    assert all(torch.equal(ys[0].view(torch.int16), y.view(torch.int16)) for y in ys[1:])
