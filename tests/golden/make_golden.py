"""Generate tests/golden/* from the UNMODIFIED reference, compiled in place
(oracle/_ref/libvidperf_ref.so, built by oracle/Makefile from
/root/reference/proj/src).  Run here, where /root/reference exists:

    make -C oracle && python tests/golden/make_golden.py

The fixtures are committed; nothing at test time reads /root/reference.
Cases restate the reference's own tests:
  * kernels_test.cpp:41-55   shift KAT (x = 100t + c, T=4, C=8, fraction 1/8)
  * kernels_test.cpp:57-61   fraction 0 is the identity
  * kernels_test.cpp:63-67   split validation (1/3 of 8, 2/3 of 9 throw; 1/3 of 9 ok)
  * kernels_test.cpp:69-84   100 seeds, shapes (1+s%2, 3+s%4, 8, 2, 3),
                             fraction 1/4 if s%3==0 else 1/8: digests of the
                             reference outputs of shift(x) and adjoint(y)
  * acceptance_test.cpp:115-166 boundary cells on ones(1,4,8,3,3)
  * BASELINE config C1       (2,8,64,56,56) fp32 from random_normal(seed), fold 8:
                             digests of x, shift(x), adjoint(x) at seeds 1 and 42
  * block cases              one residual-shift bottleneck unit (expand_layer,
                             arch.cpp:278-323) fwd+bwd through vref_block, as npz
"""
from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
from oracle.oracle import Port, Reference, ValidationError  # noqa: E402

OUT = Path(__file__).resolve().parent


def fnv(P, a):
    return f"{P.fnv1a64(np.ascontiguousarray(a)):016x}"


BLOCK_CASES = [
    # name, (N,T,C,H,W), c_out, stride, shift
    ("res2_like_identity", (1, 4, 32, 6, 6), 32, 1, (1, 8)),
    ("res2_first_projection", (2, 3, 16, 5, 5), 32, 1, (1, 8)),
    ("strided_projection", (1, 4, 32, 7, 7), 64, 2, (1, 8)),
    ("no_shift", (1, 4, 32, 6, 6), 32, 1, (0, 1)),
]


def block_weights(R, cin, c_out, stride, seed):
    """Kaiming-normal weights / N(0, 0.1) biases as init_conv does
    (net.cpp:14-22), drawn from the reference RNG with distinct seeds."""
    width = c_out // 4
    shapes = [(width, cin, 1, 1, 1), (width, width, 1, 3, 3), (c_out, width, 1, 1, 1)]
    if stride != 1 or cin != c_out:
        shapes.append((c_out, cin, 1, 1, 1))
    ws = []
    for i, s in enumerate(shapes):
        fan_in = s[1] * s[2] * s[3] * s[4]
        w = R.random_normal((1, 1, 1, 1, int(np.prod(s))), seed + 2 * i, np.sqrt(2.0 / fan_in))
        b = R.random_normal((1, 1, 1, 1, s[0]), seed + 2 * i + 1, 0.1)
        ws += [w.reshape(s), b.reshape(-1)]
    if len(ws) == 6:
        ws += [None, None]
    return ws


def main():
    R, P = Reference(), Port()
    g = {"generator": "tests/golden/make_golden.py", "source": "oracle/_ref (reference built in place)"}

    # kernels_test.cpp:41-55
    x = np.zeros((1, 4, 8, 1, 1))
    for t in range(4):
        for c in range(8):
            x[0, t, c, 0, 0] = 100.0 * t + c
    g["kat_shift"] = {"x": x.ravel().tolist(),
                      "y": R.temporal_shift(x, (1, 8)).ravel().tolist(),
                      "adjoint": R.temporal_shift_adjoint(x, (1, 8)).ravel().tolist(),
                      "shape": [1, 4, 8, 1, 1], "fraction": [1, 8]}

    # kernels_test.cpp:63-67
    val = []
    for (num, den, ch) in [(1, 3, 8), (2, 3, 9), (1, 3, 9), (1, 8, 64), (1, 8, 60), (-1, 8, 64),
                           (1, 2, 64), (3, 4, 64), (0, 1, 7), (5, 8, 8)]:
        try:
            R.validate_shift(ch, (num, den))
            ok = True
        except ValidationError:
            ok = False
        val.append({"num": num, "den": den, "channels": ch, "ok": ok})
    g["validate"] = val

    # kernels_test.cpp:69-84
    seeds = []
    for seed in range(100):
        s = (1 + seed % 2, 3 + seed % 4, 8, 2, 3)
        frac = (1, 4) if seed % 3 == 0 else (1, 8)
        xs = R.random_normal(s, seed * 2 + 1)
        ys = R.random_normal(s, seed * 2 + 2)
        seeds.append({"seed": seed, "shape": list(s), "fraction": list(frac),
                      "shift_x": fnv(P, R.temporal_shift(xs, frac)),
                      "shift_x_serial": fnv(P, R.temporal_shift(xs, frac, serial=True)),
                      "adjoint_y": fnv(P, R.temporal_shift_adjoint(ys, frac))})
    g["seed_sweep"] = seeds

    # acceptance_test.cpp:115-166 boundary cells
    ones = np.ones((1, 4, 8, 3, 3))
    sh = R.temporal_shift(ones, (1, 8))
    g["boundary"] = {"y_0_0_0": sh[0, 0, 0, 0, 0], "y_0_3_1": sh[0, 3, 1, 0, 0],
                     "y_0_1_0": sh[0, 1, 0, 0, 0], "y_0_0_2": sh[0, 0, 2, 0, 0]}

    # Config C1 digests, fp32.
    c1 = {}
    for seed in (1, 42):
        x32 = R.random_normal((2, 8, 64, 56, 56), seed).astype(np.float32)
        x64 = x32.astype(np.float64)
        c1[str(seed)] = {
            "x_f32": fnv(P, x32),
            "shift_f32": fnv(P, R.temporal_shift(x64, (1, 8), serial=True).astype(np.float32)),
            "adjoint_f32": fnv(P, R.temporal_shift_adjoint(x64, (1, 8)).astype(np.float32)),
        }
    g["c1"] = c1
    (OUT / "shift_golden.json").write_text(json.dumps(g, indent=1) + "\n")

    # Block fwd/bwd fixtures.
    arrays = {}
    meta = []
    for i, (name, shape, c_out, stride, shift) in enumerate(BLOCK_CASES):
        x = R.random_normal(shape, 700 + i)
        ws = block_weights(R, shape[2], c_out, stride, 800 + 10 * i)
        y = R.block(x, ws, c_out, stride, shift)
        gy = R.random_normal(y.shape, 900 + i)
        y2, gx, gws = R.block(x, ws, c_out, stride, shift, gy=gy)
        assert np.array_equal(y, y2)
        arrays[f"{name}/x"] = x
        arrays[f"{name}/gy"] = gy
        arrays[f"{name}/y"] = y
        arrays[f"{name}/gx"] = gx
        for j, (w, gw) in enumerate(zip(ws, gws)):
            if w is not None:
                arrays[f"{name}/w{j}"] = w
                arrays[f"{name}/gw{j}"] = gw
        meta.append({"name": name, "shape": list(shape), "c_out": c_out, "stride": stride,
                     "shift": list(shift)})
    np.savez_compressed(OUT / "block_golden.npz", **arrays)
    (OUT / "block_golden.json").write_text(json.dumps(meta, indent=1) + "\n")
    print("wrote", sorted(p.name for p in OUT.iterdir()))


if __name__ == "__main__":
    main()
