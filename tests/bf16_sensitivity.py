"""TEST-ONLY analysis: how far do TSM-R50 gradients move when only the
operand/storage precision changes?  Runs the reference algorithm in fp64
(torch, CPU) on the reference's own weights (vidperf::Network(build_tsm8f()
at HW x HW, 42), input random_normal seed 43; ref_capi.cpp) three ways:

  exact      fp64 everywhere (= Network::loss_gradients up to summation order)
  wx         weights and input rounded to bf16 once (what a bf16 tensor-core
             path computes on), everything else fp64
  act        stored activations rounded to bf16 (conv outputs, pool output,
             block outputs), weights/input exact
  all        both, plus bf16-rounded stored gradients (the B200 path's
             storage precision)

and prints the per-tensor rel-L2 of each against `exact`.  The B200 network
(bf16 operands, fp32 accumulation) matches `all` (tests/test_network_gpu.py
prints its own errors): conv1.w and the input gradient are intrinsically
sensitive — rounding only the weights and the input to bf16 already moves
conv1.w by ~12% at 64x64 — because max-pool argmax and ReLU decisions near
ties flip and reroute whole gradient elements.  This is why the network
tests bound those two tensors separately.

    python tests/bf16_sensitivity.py [HW] [N]
"""
import sys
from pathlib import Path

import numpy as np
import torch
import torch.nn.functional as F

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))


def main(hw=64, n=2):
    from oracle.oracle import Reference
    import torch_tsm_ref as T
    torch.set_default_dtype(torch.float64)
    R = Reference()
    flat = torch.from_numpy(R.net_sized(hw, hw, 42).param_vector())
    x0 = torch.from_numpy(R.random_normal((n, 8, 3, hw, hw), 43))
    shapes, names = [(64, 3, 7, 7), (64,)], ["conv1.w", "conv1.b"]
    cin = 64
    for s, (blocks, cout) in enumerate(zip((3, 4, 6, 3), (256, 512, 1024, 2048))):
        for bi in range(blocks):
            stride = 2 if (s > 0 and bi == 0) else 1
            w = cout // 4
            shapes += [(w, cin, 1, 1), (w,), (w, w, 3, 3), (w,), (cout, w, 1, 1), (cout,)]
            names += [f"res{s + 2}.{bi}.{k}" for k in ("w1", "b1", "w2", "b2", "w3", "b3")]
            if stride != 1 or cin != cout:
                shapes += [(cout, cin, 1, 1), (cout,)]
                names += [f"res{s + 2}.{bi}.wp", f"res{s + 2}.{bi}.bp"]
            cin = cout
    shapes += [(400, 2048, 1, 1), (400,)]
    names += ["fc.w", "fc.b"]

    def bf(a):
        return a.float().bfloat16().double()

    mode = {}

    class RB(torch.autograd.Function):
        @staticmethod
        def forward(ctx, a):
            return bf(a)

        @staticmethod
        def backward(ctx, g):
            return bf(g) if mode["grad"] else g

    def run(wx, act, grad):
        mode["grad"] = grad
        rw = RB.apply if wx else (lambda a: a)
        ra = RB.apply if act else (lambda a: a)
        params, pos = [], 0
        for sh in shapes:
            k = int(np.prod(sh))
            params.append(flat[pos:pos + k].reshape(sh).clone().requires_grad_(True))
            pos += k
        P = [rw(p) if p.dim() > 1 else p for p in params]
        x = x0.clone().requires_grad_(True)
        h = F.conv2d(rw(x).reshape(n * 8, 3, hw, hw), P[0], P[1], stride=2, padding=3)
        h = ra(F.max_pool2d(ra(h), 3, 2, 1))
        it, cin = iter(P[2:]), 64
        for s, (blocks, cout) in enumerate(zip((3, 4, 6, 3), (256, 512, 1024, 2048))):
            for bi in range(blocks):
                stride = 2 if (s > 0 and bi == 0) else 1
                a1, c1, a2, c2, a3, c3 = [next(it) for _ in range(6)]
                r = ra(F.relu(F.conv2d(T.shift(h, n, 8, cin // 8), a1, c1)))
                r = ra(F.relu(F.conv2d(r, a2, c2, stride=stride, padding=1)))
                r = F.conv2d(r, a3, c3)
                if stride != 1 or cin != cout:
                    ap, cp = next(it), next(it)
                    sk = ra(F.conv2d(h, ap, cp, stride=stride))
                else:
                    sk = h
                h = ra(F.relu(r + sk))
                cin = cout
        feat = h.reshape(n, 8, *h.shape[1:]).mean(dim=(1, 3, 4))
        wf, bfc = next(it), next(it)
        y = F.linear(feat, wf.reshape(400, -1), bfc)
        (y ** 2).sum().backward()
        return [p.grad.clone() for p in params] + [x.grad.clone()]

    exact = run(False, False, False)
    rel = lambda a, b: float((a - b).norm() / b.norm())  # noqa: E731
    print(f"TSM-R50 {n}x{hw}x{hw}, reference weights (seed 42) and input (seed 43); "
          "rel-L2 of each gradient against fp64:")
    rows = {}
    for label, cfg in (("wx", (True, False, False)), ("act", (False, True, False)),
                       ("all", (True, True, True))):
        g = run(*cfg)
        rows[label] = [rel(a, b) for a, b in zip(g, exact)]
    print(f"{'tensor':14s} {'wx':>9s} {'act':>9s} {'all':>9s}")
    for i, nm in enumerate(names + ["input"]):
        if nm in ("conv1.w", "conv1.b", "input", "res2.0.w1", "fc.w") or i == len(names):
            print(f"{nm:14s} " + " ".join(f"{rows[k][i]:9.3e}" for k in ("wx", "act", "all")))
    for k in ("wx", "act", "all"):
        params = rows[k][:-1]
        print(f"{k:4s}: parameter tensors median {np.median(params):.3e}, worst "
              f"{names[int(np.argmax(params))]} {max(params):.3e}, second "
              f"{sorted(params)[-2]:.3e}; input {rows[k][-1]:.3e}")


if __name__ == "__main__":
    main(*(int(a) for a in sys.argv[1:]))
