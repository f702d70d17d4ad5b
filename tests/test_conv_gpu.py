"""GPU numerics of the tcgen05 conv engine against a plain fp32 torch
reference of the same op on the same bf16-rounded inputs."""
import numpy as np
import pytest
import torch

from paper_1910_00932_b200 import conv

pytestmark = pytest.mark.gpu


def shift_ref(x, f, b):
    """Reference temporal shift on NTHWC (kernels.cpp:97-125): channels [0,f)
    from t-1, [f,f+b) from t+1, zero at the clip boundary."""
    y = x.clone()
    y[:, :, ..., :f + b] = 0
    if f:
        y[:, 1:, ..., :f] = x[:, :-1, ..., :f]
    if b:
        y[:, :-1, ..., f:f + b] = x[:, 1:, ..., f:f + b]
    return y


def rel_err(got, want):
    return float((got.float() - want).abs().max() / want.abs().max().clamp_min(1e-30))


@pytest.mark.parametrize("n,t,h,w,cin,cout,f", [
    (1, 4, 6, 6, 64, 64, 8),       # F=8 at 64 channels: three-frame tile kernel
    (2, 8, 17, 9, 64, 64, 8),      # ... partial 16 x 8 tiles, 8 frames
    (3, 1, 5, 5, 64, 64, 8),       # ... one frame per clip: both groups zero
    (2, 8, 14, 14, 256, 64, 32),   # res2 conv1 shape (small HW), KC=32
    (1, 8, 7, 7, 512, 128, 64),    # KC=64, partial tail tile
    (2, 3, 5, 5, 64, 256, 0),      # no shift (conv3-like)
    (1, 8, 28, 28, 1024, 256, 128),
    (1, 2, 4, 4, 128, 512, 16),    # F=16 -> KC=8 path (16 % 32 != 0)
])
@pytest.mark.parametrize("relu", [False, True])
def test_conv1x1_fused_shift(n, t, h, w, cin, cout, f, relu):
    torch.manual_seed(0)
    dev = torch.device("cuda")
    x = torch.randn(n, t, h, w, cin, device=dev).bfloat16()
    wt = (torch.randn(cout, cin, device=dev) / cin ** 0.5).bfloat16()
    b = torch.randn(cout, device=dev) * 0.1
    y = conv.conv1x1_fwd(x, wt, b, fold=(f, f), relu=relu)
    ref = shift_ref(x.float(), f, f) @ wt.float().t() + b
    if relu:
        ref = ref.clamp_min(0)
    torch.cuda.synchronize()
    assert rel_err(y, ref) < 1e-2, rel_err(y, ref)


@pytest.mark.parametrize("fold", [(8, 0), (0, 8), (16, 0), (8, 8)])
@pytest.mark.parametrize("t", [1, 2, 8])
def test_shift1x1_c64_groups(fold, t):
    """The three-frame tile kernel (64 -> 64 channels, F + B <= 16) for
    asymmetric groups and short clips, against the shifted fp32 GEMM."""
    torch.manual_seed(5)
    dev = torch.device("cuda")
    x = torch.randn(2, t, 9, 11, 64, device=dev).bfloat16()
    wt = (torch.randn(64, 64, device=dev) / 8).bfloat16()
    b = torch.randn(64, device=dev) * 0.1
    y = conv.conv1x1_fwd(x, wt, b, fold=fold, relu=True)
    ref = (shift_ref(x.float(), *fold) @ wt.float().t() + b).clamp_min(0)
    assert rel_err(y, ref) < 1e-2, rel_err(y, ref)


@pytest.mark.parametrize("cin,cout", [
    (64, 256),     # 1 k-block: residual as identity k-blocks (res2 conv3)
    (256, 1024),   # 4 k-blocks, 4 N tiles: identity blocks per N tile (res4 conv3)
    (512, 2048),   # 8 k-blocks (res5 conv3)
    (1024, 256),   # 16 k-blocks: residual added in the epilogue
])
def test_conv1x1_residual_relu(cin, cout):
    torch.manual_seed(1)
    dev = torch.device("cuda")
    x = torch.randn(2, 4, 7, 9, cin, device=dev).bfloat16()
    wt = (torch.randn(cout, cin, device=dev) / cin ** 0.5).bfloat16()
    b = torch.randn(cout, device=dev) * 0.1
    r = torch.randn(2, 4, 7, 9, cout, device=dev).bfloat16()
    y = conv.conv1x1_fwd(x, wt, b, relu=True, residual=r)
    ref = (x.float() @ wt.float().t() + b + r.float()).clamp_min(0)
    assert rel_err(y, ref) < 1e-2


# ---------------------------------------------------------------------------
# kxk / strided forward, dgrad, wgrad against torch fp32 on the same bf16 data

import torch.nn.functional as Fnn  # noqa: E402


def nchw(x):  # NTHWC -> (N*T, C, H, W) fp32
    n, t, h, w, c = x.shape
    return x.float().reshape(n * t, h, w, c).permute(0, 3, 1, 2)


def nthwc(y, n, t):  # (N*T, C, H, W) -> NTHWC
    f, c, h, w = y.shape
    return y.permute(0, 2, 3, 1).reshape(n, t, h, w, c)


CONV_CASES = [
    # n, t, h, w, cin, cout, k, stride
    (1, 4, 6, 6, 64, 64, 3, 1),
    (2, 2, 8, 8, 128, 64, 3, 2),
    (1, 3, 7, 7, 256, 256, 3, 1),
    (1, 2, 14, 14, 64, 128, 1, 2),   # strided projection (im2col 1x1)
    (1, 2, 5, 9, 64, 64, 3, 1),      # non-square
]


@pytest.mark.parametrize("case", CONV_CASES)
def test_conv_kxk_fwd(case):
    n, t, h, w, cin, cout, k, s = case
    torch.manual_seed(2)
    x = torch.randn(n, t, h, w, cin, device="cuda").bfloat16()
    wt = (torch.randn(cout, k, k, cin, device="cuda") / (k * (cin ** 0.5))).bfloat16()
    b = torch.randn(cout, device="cuda") * 0.1
    y = conv.conv_fwd(x, wt, b, k=k, stride=s, relu=True)
    ref = Fnn.conv2d(nchw(x), wt.float().permute(0, 3, 1, 2), b, stride=s, padding=k // 2)
    ref = nthwc(ref.clamp_min(0), n, t)
    assert rel_err(y, ref) < 1e-2


@pytest.mark.parametrize("case", CONV_CASES)
def test_conv_kxk_dgrad_wgrad(case):
    n, t, h, w, cin, cout, k, s = case
    torch.manual_seed(3)
    x = torch.randn(n, t, h, w, cin, device="cuda").bfloat16()
    wm = torch.randn(cout, k, k, cin, device="cuda") / (k * (cin ** 0.5))
    wf, wd = conv.weights_to_bf16(wm)
    ho, wo = conv.out_hw(h, w, k, s)
    dy = torch.randn(n, t, ho, wo, cout, device="cuda").bfloat16()
    # torch reference gradients in fp32
    xr = nchw(x).requires_grad_(True)
    wr = wf.float().reshape(cout, k, k, cin).permute(0, 3, 1, 2).contiguous().requires_grad_(True)
    yr = Fnn.conv2d(xr, wr, None, stride=s, padding=k // 2)
    yr.backward(nchw(dy))
    dx = conv.conv_dgrad(dy, wd, x.shape, k=k, stride=s)
    dw = conv.conv_wgrad(x, dy, k=k, stride=s)
    assert rel_err(dx, nthwc(xr.grad, n, t)) < 1e-2
    assert rel_err(dw, wr.grad.permute(0, 2, 3, 1)) < 1e-2


@pytest.mark.parametrize("case", [
    # n, t, h, w, cin, cout — 3x3 stride 2 (sub-pixel parity classes)
    (2, 2, 28, 28, 128, 128),   # 784 dY pixels: ragged last M tile
    (1, 3, 14, 14, 256, 256),   # BN 256
    (1, 2, 56, 56, 64, 128),    # BN 64
    (1, 1, 2, 2, 64, 64),       # single dY pixel
])
def test_dgrad_strided3x3_subpixel_mask_residual(case):
    n, t, h, w, cin, cout = case
    torch.manual_seed(11)
    wm = torch.randn(cout, 3, 3, cin, device="cuda") / (3 * (cin ** 0.5))
    wf, wd = conv.weights_to_bf16(wm)
    dy = torch.randn(n, t, h // 2, w // 2, cout, device="cuda").bfloat16()
    res = torch.randn(n, t, h, w, cin, device="cuda").bfloat16()
    mask = torch.randn(n, t, h, w, cin, device="cuda").clamp_min(0).bfloat16()
    xr = torch.zeros(n * t, cin, h, w, device="cuda", requires_grad=True)
    wr = wf.float().reshape(cout, 3, 3, cin).permute(0, 3, 1, 2)
    Fnn.conv2d(xr, wr, None, stride=2, padding=1).backward(nchw(dy))
    ref = (nthwc(xr.grad, n, t) + res.float()) * (mask.float() > 0)
    dx = conv.conv_dgrad(dy, wd, (n, t, h, w, cin), k=3, stride=2, residual=res, mask=mask)
    assert rel_err(dx, ref) < 1e-2
    # every dx element written (no stale memory): compare against a poisoned buffer
    out = torch.full((n, t, h, w, cin), float("nan"), device="cuda").bfloat16()
    dx2 = conv.conv_dgrad(dy, wd, (n, t, h, w, cin), k=3, stride=2, residual=res, mask=mask,
                          out=out)
    assert torch.equal(dx2, dx)


@pytest.mark.parametrize("c", [64, 128])
@pytest.mark.parametrize("hw", [(56, 56), (28, 28), (7, 7), (17, 9)])
def test_halo3x3_c64(hw, c):
    # 64 -> 64, 3x3, stride 1: the halo-tile kernels (forward, dgrad + mask,
    # wgrad + fused bias grad through the all-ones MMA rows); 128 -> 128: the
    # streamed-weight halo kernel (forward, unmasked dgrad) and the im2col wgrad
    h, w = hw
    n, t = 2, 2
    torch.manual_seed(12)
    x = torch.randn(n, t, h, w, c, device="cuda").bfloat16()
    wm = torch.randn(c, 3, 3, c, device="cuda") / (3 * 8)
    wf, wd = conv.weights_to_bf16(wm)
    b = torch.randn(c, device="cuda") * 0.1
    wr = wf.float().reshape(c, 3, 3, c).permute(0, 3, 1, 2).contiguous()
    y = conv.conv_fwd(x, wf, b, k=3, relu=True)
    ref = nthwc(Fnn.conv2d(nchw(x), wr, b, padding=1).clamp_min(0), n, t)
    assert rel_err(y, ref) < 1e-2
    dy = torch.randn(n, t, h, w, c, device="cuda").bfloat16()
    mask = torch.randn(n, t, h, w, c, device="cuda").clamp_min(0).bfloat16()
    xr = nchw(x).requires_grad_(True)
    wrg = wr.clone().requires_grad_(True)
    Fnn.conv2d(xr, wrg, None, padding=1).backward(nchw(dy))
    dx = conv.conv_dgrad(dy, wd, x.shape, k=3, mask=mask)
    assert rel_err(dx, nthwc(xr.grad, n, t) * (mask.float() > 0)) < 1e-2
    dx_nomask = conv.conv_dgrad(dy, wd, x.shape, k=3)
    assert rel_err(dx_nomask, nthwc(xr.grad, n, t)) < 1e-2
    dw, db = conv.conv_wgrad(x, dy, k=3, bias_grad=True)
    assert rel_err(dw, wrg.grad.permute(0, 2, 3, 1)) < 1e-2
    assert rel_err(db, dy.float().sum(dim=(0, 1, 2, 3))) < 1e-4
    # deterministic: bitwise identical on a second run
    dw2, db2 = conv.conv_wgrad(x, dy, k=3, bias_grad=True)
    assert torch.equal(dw, dw2) and torch.equal(db, db2)


_HALO_DIGEST = """
import sys, hashlib, torch
sys.path.insert(0, {root!r})
from paper_1910_00932_b200 import conv
torch.manual_seed(21)
c = {c}
h = hashlib.sha256()
for n, t, hh, ww in ((1, 3, 7, 7), (1, 3, 28, 28), (2, 1, 17, 9)):
    x = torch.randn(n, t, hh, ww, c, device="cuda").bfloat16()
    wf, wd = conv.weights_to_bf16(torch.randn(c, 3, 3, c, device="cuda") / (3 * c ** 0.5))
    b = torch.randn(c, device="cuda") * 0.1
    mask = torch.randn(n, t, hh, ww, c, device="cuda").clamp_min(0).bfloat16()
    y = conv.conv_fwd(x, wf, b, k=3, relu=True)
    dx = conv.conv_dgrad(x, wd, x.shape, k=3)
    dxm = conv.conv_dgrad(x, wd, x.shape, k=3, mask=mask) if c == 64 else dx
    torch.cuda.synchronize()
    for r in (y, dx, dxm):
        h.update(r.float().cpu().numpy().tobytes())
print(h.hexdigest())
"""


_SUBPIX_DIGEST = """
import sys, hashlib, torch
sys.path.insert(0, {root!r})
from paper_1910_00932_b200 import conv
torch.manual_seed(23)
h = hashlib.sha256()
for n, t, ho, c in ((1, 3, 14, 128), (2, 2, 14, 256), (1, 5, 7, 512), (1, 1, 7, 128)):
    dy = torch.randn(n, t, ho, ho, c, device="cuda").bfloat16()
    _, wd = conv.weights_to_bf16(torch.randn(c, 3, 3, c, device="cuda") / (3 * c ** 0.5))
    dx = conv.conv_dgrad(dy, wd, (n, t, 2 * ho, 2 * ho, c), k=3, stride=2)
    torch.cuda.synchronize()
    h.update(dx.float().cpu().numpy().tobytes())
print(h.hexdigest())
"""


def test_subpix_tma_bitwise_equals_thread_scatter():
    """The merged sub-pixel dgrad with row-aligned tiles stored through the
    5-D class map (TSM_SUBPIX_TMA=1, default where the tiles keep >= 120
    rows: 14 / 7-wide class grids) gives bitwise the per-thread scatter's dx
    (=0): partial last tiles, odd tile counts, CTA pairs at 256 / 512
    channels; two processes."""
    import os
    import subprocess
    import sys
    from pathlib import Path
    code = _SUBPIX_DIGEST.format(root=str(Path(__file__).resolve().parents[1]))
    digests = []
    for v in ("1", "0"):
        r = subprocess.run([sys.executable, "-c", code], env=dict(os.environ, TSM_SUBPIX_TMA=v),
                           capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stderr[-3000:]
        digests.append(r.stdout.strip().splitlines()[-1])
    assert digests[0] == digests[1]


@pytest.mark.parametrize("switch,c,modes", [("TSM_HALO128", 128, ("2", "1"))])
def test_halo_pair_bitwise_equals_single(switch, c, modes):
    """The 128-channel 3x3 halo kernel on CTA pairs (default) and on single
    CTAs gives bitwise the same forward and input gradient, including odd
    tile counts (a padding tile in the last pair); two processes, one per
    path."""
    import os
    import subprocess
    import sys
    from pathlib import Path
    code = _HALO_DIGEST.format(root=str(Path(__file__).resolve().parents[1]), c=c)
    digests = []
    for v in modes:
        r = subprocess.run([sys.executable, "-c", code], env=dict(os.environ, **{switch: v}),
                           capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stderr[-3000:]
        digests.append(r.stdout.strip().splitlines()[-1])
    assert digests[0] == digests[1]


@pytest.mark.parametrize("case", [
    (2, 4, 5, 5, 64, 128, 8),       # narrow split: epilogue residual
    (2, 8, 6, 6, 1024, 256, 128),   # skip gradient as identity k-blocks, 4 N tiles
])
def test_dgrad_shift_adjoint_fused(case):
    torch.manual_seed(4)
    n, t, h, w, cin, cout, f = case
    dy = torch.randn(n, t, h, w, cout, device="cuda").bfloat16()
    wm = torch.randn(cout, 1, 1, cin, device="cuda") / 8
    wf, wd = conv.weights_to_bf16(wm)
    res = torch.randn(n, t, h, w, cin, device="cuda").bfloat16()
    mask = torch.randn(n, t, h, w, cin, device="cuda").bfloat16()
    dx = conv.conv_dgrad(dy, wd, (n, t, h, w, cin), fold=(f, f), residual=res, mask=mask)
    g = dy.float() @ wf.float()  # dgrad before the adjoint shift
    adj = torch.zeros_like(g)
    adj[:, :-1, ..., :f] = g[:, 1:, ..., :f]          # c < F reads t+1
    adj[:, 1:, ..., f:2 * f] = g[:, :-1, ..., f:2 * f]  # F <= c < 2F reads t-1
    adj[..., 2 * f:] = g[..., 2 * f:]
    ref = (adj + res.float()) * (mask.float() > 0)
    assert rel_err(dx, ref) < 1e-2


@pytest.mark.parametrize("case", [
    (2, 8, 17, 9, (8, 8), True),    # res2.0: partial 16 x 8 tiles, skip gradient
    (1, 1, 5, 5, (8, 8), True),     # one frame per clip: both groups vanish
    (2, 3, 6, 6, (16, 0), False),   # one group, no skip
    (1, 4, 7, 7, (0, 8), True),
])
def test_dgrad_shift_adjoint_c64(case):
    """64 -> 64 adjoint shift + skip on the three-frame tile kernel (masked
    dgrad weights per source frame), against the fp32 adjoint."""
    torch.manual_seed(4)
    n, t, h, w, (fa, fb), with_res = case
    dy = torch.randn(n, t, h, w, 64, device="cuda").bfloat16()
    wf, wd = conv.weights_to_bf16(torch.randn(64, 1, 1, 64, device="cuda") / 8)
    res = torch.randn(n, t, h, w, 64, device="cuda").bfloat16() if with_res else None
    dx = conv.conv_dgrad(dy, wd, (n, t, h, w, 64), fold=(fa, fb), residual=res)
    g = dy.float() @ wf.float()
    adj = g.clone()
    adj[..., :fa + fb] = 0
    adj[:, :-1, ..., :fa] = g[:, 1:, ..., :fa]                    # c < F reads t+1
    adj[:, 1:, ..., fa:fa + fb] = g[:, :-1, ..., fa:fa + fb]      # F <= c < F+B reads t-1
    ref = adj + (res.float() if with_res else 0)
    assert rel_err(dx, ref) < 1e-2, rel_err(dx, ref)


@pytest.mark.parametrize("f", [8, 16, 32, 64])  # 8, 16: virtual channels (conv_wgrad_vshift)
def test_wgrad_shifted_x(f):
    torch.manual_seed(5)
    n, t, h, w, cin, cout = 2, 4, 6, 6, 8 * f, 64
    x = torch.randn(n, t, h, w, cin, device="cuda").bfloat16()
    dy = torch.randn(n, t, h, w, cout, device="cuda").bfloat16()
    dw = conv.conv_wgrad(x, dy, fold=(f, f))
    xs = shift_ref(x.float(), f, f)
    ref = dy.float().reshape(-1, cout).t() @ xs.reshape(-1, cin)
    assert rel_err(dw.reshape(cout, cin), ref) < 1e-2


@pytest.mark.parametrize("case", [
    (2, 8, 17, 9, (8, 8)),     # res2.0 split, partial 8 x 8 patches
    (1, 1, 5, 5, (8, 8)),      # one frame per clip: shifted groups see zeros
    (3, 3, 8, 8, (16, 0)),
    (1, 4, 7, 6, (0, 8)),
])
def test_wgrad_shift1_c64(case):
    """64 -> 64 weight and bias gradient of the narrow-split shifted 1x1 on
    the three-frame patch kernel, against fp32; deterministic (bitwise
    equal on a second run)."""
    torch.manual_seed(7)
    n, t, h, w, fold = case
    x = torch.randn(n, t, h, w, 64, device="cuda").bfloat16()
    dy = torch.randn(n, t, h, w, 64, device="cuda").bfloat16()
    dw, db = conv.conv_wgrad(x, dy, fold=fold, bias_grad=True)
    xs = shift_ref(x.float(), *fold)
    ref = dy.float().reshape(-1, 64).t() @ xs.reshape(-1, 64)
    assert rel_err(dw.reshape(64, 64), ref) < 1e-2
    assert rel_err(db, dy.float().sum(dim=(0, 1, 2, 3))) < 1e-4
    dw2, db2 = conv.conv_wgrad(x, dy, fold=fold, bias_grad=True)
    assert torch.equal(dw, dw2) and torch.equal(db, db2)


@pytest.mark.parametrize("case", [
    (4, 8, 28, 28, 256, 64, 32),     # res2.1-like at 4 clips: split-K over many chunks
    (3, 8, 14, 14, 512, 128, 64),    # uneven last chunk, 128 output channels
    (2, 8, 7, 7, 1024, 256, 128),    # clip remainders gathered at the K end
])
def test_wgrad_shifted_interleaved_splitk(case):
    """Shifted-x weight gradient with the split-K chunks interleaved over the
    splits (TSM_WGRAD_ILV, default 4 k-blocks): against fp32, deterministic
    on a second run, and the bias gradient from the same pass."""
    torch.manual_seed(8)
    n, t, h, w, cin, cout, f = case
    x = torch.randn(n, t, h, w, cin, device="cuda").bfloat16()
    dy = torch.randn(n, t, h, w, cout, device="cuda").bfloat16()
    dw, db = conv.conv_wgrad(x, dy, fold=(f, f), bias_grad=True)
    xs = shift_ref(x.float(), f, f)
    ref = dy.float().reshape(-1, cout).t() @ xs.reshape(-1, cin)
    assert rel_err(dw.reshape(cout, cin), ref) < 1e-2
    assert rel_err(db, dy.float().sum(dim=(0, 1, 2, 3))) < 1e-4
    dw2, db2 = conv.conv_wgrad(x, dy, fold=(f, f), bias_grad=True)
    assert torch.equal(dw, dw2) and torch.equal(db, db2)


def test_bias_grad_and_layout():
    torch.manual_seed(6)
    g = torch.randn(3, 4, 7, 7, 256, device="cuda").bfloat16()
    db = conv.bias_grad(g)
    assert rel_err(db, g.float().sum(dim=(0, 1, 2, 3))) < 1e-4
    x = torch.randn(2, 3, 24, 5, 7, device="cuda")
    y = conv.to_nthwc(x, c_pad=32)
    assert torch.equal(y[..., :24].float(), x.bfloat16().float().permute(0, 1, 3, 4, 2))
    assert (y[..., 24:] == 0).all()
    back = conv.to_ntchw(y[..., :24].contiguous(), torch.float32)
    assert torch.equal(back, x.bfloat16().float())


def test_conv7x7_c8_forward():
    # 7x7 / stride 2 / pad 3 on 8-channel pixels (16-byte rows, unswizzled
    # KC=8 slabs); K = 49*8 = 392 is zero-padded to 448 in the weights.  (The
    # network's conv1 uses a materialised im2col matrix instead, covered by
    # tests/test_network_gpu.py.)  The im2col weight gradient needs c_in % 64.
    torch.manual_seed(7)
    n, t, h, w, cout = 1, 2, 40, 36, 64
    x = torch.zeros(n, t, h, w, 8, device="cuda")
    x[..., :3] = torch.randn(n, t, h, w, 3, device="cuda")
    x = x.bfloat16()
    wm = torch.zeros(cout, 7, 7, 8, device="cuda")
    wm[..., :3] = torch.randn(cout, 7, 7, 3, device="cuda") / 10
    wf, _ = conv.weights_to_bf16(wm, k_pad=448, dgrad=False)
    b = torch.randn(cout, device="cuda") * 0.1
    y = conv.conv_fwd(x, wf, b, k=7, stride=2)
    wr = wf[:, :392].float().reshape(cout, 7, 7, 8).permute(0, 3, 1, 2).contiguous()
    ref = Fnn.conv2d(nchw(x), wr, b, stride=2, padding=3)
    assert rel_err(y, nthwc(ref, n, t)) < 1e-2
    with pytest.raises(NotImplementedError):
        conv.conv_wgrad(x, torch.zeros_like(y), k=7, stride=2)


@pytest.mark.parametrize("f,hw", [(32, (6, 6)), (64, (28, 28)), (32, (7, 7))])
def test_dgrad_shift_adjoint_tma_path(f, hw):
    # F % 32 == 0: the TMA epilogue (row-offset stores, direct stores above
    # the clip start, boundary-frame fixup kernel).
    torch.manual_seed(8)
    n, t, cout = 2, 4, 64
    h, w = hw
    cin = 8 * f
    dy = torch.randn(n, t, h, w, cout, device="cuda").bfloat16()
    wm = torch.randn(cout, 1, 1, cin, device="cuda") / 8
    wf, wd = conv.weights_to_bf16(wm)
    res = torch.randn(n, t, h, w, cin, device="cuda").bfloat16()
    mask = torch.randn(n, t, h, w, cin, device="cuda").bfloat16()
    dx = conv.conv_dgrad(dy, wd, (n, t, h, w, cin), fold=(f, f), residual=res, mask=mask)
    g = dy.float() @ wf.float()
    adj = torch.zeros_like(g)
    adj[:, :-1, ..., :f] = g[:, 1:, ..., :f]
    adj[:, 1:, ..., f:2 * f] = g[:, :-1, ..., f:2 * f]
    adj[..., 2 * f:] = g[..., 2 * f:]
    ref = (adj + res.float()) * (mask.float() > 0)
    assert rel_err(dx, ref) < 1e-2


@pytest.mark.parametrize("case", [
    (2, 4, 6, 6, 256, 64, 1, 1, 32),    # swapped wgrad (c_out 64), shifted x
    (2, 8, 14, 14, 64, 64, 1, 1, 8),    # narrow split in virtual channels (res2.0)
    (1, 8, 7, 7, 512, 256, 1, 1, 0),    # A-operand dY (c_out >= 128)
    (1, 4, 8, 8, 64, 64, 3, 1, 0),      # swapped, im2col
    (1, 4, 8, 8, 128, 128, 3, 2, 0),    # strided 3x3, A-operand dY
])
def test_wgrad_fused_bias_grad(case):
    n, t, h, w, cin, cout, k, s, f = case
    torch.manual_seed(9)
    x = torch.randn(n, t, h, w, cin, device="cuda").bfloat16()
    ho, wo = conv.out_hw(h, w, k, s)
    dy = torch.randn(n, t, ho, wo, cout, device="cuda").bfloat16()
    dw, db = conv.conv_wgrad(x, dy, k=k, stride=s, fold=(f, f), bias_grad=True)
    assert rel_err(db, dy.float().sum(dim=(0, 1, 2, 3))) < 1e-4
    dw2 = conv.conv_wgrad(x, dy, k=k, stride=s, fold=(f, f))
    assert torch.equal(dw, dw2)


def maxpool_ref(x):
    """max_pool_forward / max_pool_backward (kernels.cpp:353-455) on NTHWC:
    1x3x3 / stride 2 / pad 1, padded taps never win, ties keep the first tap
    in (h, w) scan order.  Returns (y, tap index 0..8, backward fn)."""
    n, t, h, w, c = x.shape
    ho, wo = (h - 1) // 2 + 1, (w - 1) // 2 + 1
    xp = torch.full((n, t, h + 2, w + 2 + 1, c), float("-inf"), device=x.device)
    xp[:, :, 1:h + 1, 1:w + 1] = x.float()
    xp = torch.cat([xp, torch.full_like(xp[:, :, :1], float("-inf"))], dim=2)
    taps = torch.stack([xp[:, :, dh:dh + 2 * ho:2, dw:dw + 2 * wo:2]
                        for dh in range(3) for dw in range(3)], dim=0)
    y, arg = taps.max(dim=0)  # first maximal index on ties
    first = torch.argmax((taps == y.unsqueeze(0)).to(torch.uint8), dim=0)

    def backward(gy):
        gx = torch.zeros(n, t, h + 3, w + 3, c, device=x.device, dtype=torch.float64)
        for k in range(9):
            dh, dw = divmod(k, 3)
            sel = (first == k).double() * gy.double()
            gx[:, :, dh:dh + 2 * ho:2, dw:dw + 2 * wo:2] += sel
        return gx[:, :, 1:h + 1, 1:w + 1]
    return y, first, backward


@pytest.mark.parametrize("shape", [(2, 8, 112, 112, 64),   # network stem (even path)
                                   (1, 3, 17, 10, 16),     # odd H: general path
                                   (1, 2, 9, 9, 8),
                                   (1, 3, 22, 14, 16),     # 2x2 bwd, partial strips
                                   (1, 2, 10, 10, 8)])     # 2x2 bwd, odd argmax row
@pytest.mark.parametrize("ties", [False, True])
def test_maxpool_fwd_bwd(shape, ties):
    torch.manual_seed(11)
    x = torch.randn(*shape, device="cuda")
    if ties:  # few distinct values: most windows have several maximal taps
        x = x.mul(1.5).round().clamp(-2, 2)
    x = x.bfloat16()
    y, arg = conv.maxpool_fwd(x)
    y_ref, arg_ref, bwd = maxpool_ref(x)
    assert torch.equal(y.float(), y_ref)
    assert torch.equal(arg.long(), arg_ref)
    gy = torch.randn_like(y.float()).bfloat16()
    gx = conv.maxpool_bwd(gy, arg, x.shape)
    want = bwd(gy.float())
    # at most 4 windows meet at a pixel: fp32 sums rounded once to bf16
    assert torch.equal(gx.float(), want.float().bfloat16().float()) or \
        float((gx.double() - want).abs().max()) <= float(want.abs().max()) * 2 ** -8


def _bits(t):
    return t.contiguous().view(torch.int16)


@pytest.mark.parametrize("shape", [(2, 8, 112, 112, 64),   # network stem (2x2-block bwd)
                                   (1, 3, 17, 10, 16),     # odd H: general bwd
                                   (1, 2, 9, 9, 8)])
@pytest.mark.parametrize("special", ["ties", "nan"])
def test_maxpool_bitexact_vs_reference(ref, shape, special):
    """max_pool_forward / max_pool_backward of the reference itself
    (kernels.cpp:353-455, via oracle/_ref) on the same bf16 values: output and
    input gradient bit for bit.  "nan": the reference's `!seen || v > best`
    keeps a NaN only when it is a window's first valid tap and never lets a
    later NaN replace the maximum; "ties": most windows have several maximal
    taps (the first in scan order wins)."""
    n, t, h, w, c = shape
    rng = np.random.default_rng(17)
    x = rng.standard_normal((n, t, c, h, w))
    if special == "ties":
        x = np.clip(np.round(x * 1.5), -2, 2)
    else:
        x[rng.random(x.shape) < 0.05] = np.nan
    xb = torch.from_numpy(x).float().bfloat16()
    gy_shape = (n, t, c, (h - 1) // 2 + 1, (w - 1) // 2 + 1)
    gy = torch.from_numpy(rng.standard_normal(gy_shape)).float().bfloat16()
    y_ref, gx_ref = ref.max_pool(xb.double().numpy(), (1, 3, 3), (1, 2, 2), (0, 1, 1),
                                 gy=gy.double().numpy())
    xd = conv.to_nthwc(xb.cuda())
    y, arg = conv.maxpool_fwd(xd)
    gx = conv.maxpool_bwd(conv.to_nthwc(gy.cuda()), arg, xd.shape)
    y_got = conv.to_ntchw(y, torch.float64).cpu().numpy()
    gx_got = conv.to_ntchw(gx, torch.float64).cpu().numpy()
    y_want = torch.from_numpy(y_ref).bfloat16().double().numpy()   # exact: y_ref is an x value
    gx_want = torch.from_numpy(gx_ref).bfloat16().double().numpy()
    assert np.array_equal(y_got, y_want, equal_nan=True)
    assert np.array_equal(gx_got, gx_want, equal_nan=True)
    if special == "nan":
        assert np.isnan(y_got).any()


@pytest.mark.parametrize("hw", [(2, 2), (3, 3), (1, 5)])
def test_dgrad_shift_adjoint_short_clips(hw):
    """Clips shorter than one 128-row tile (T*H*W < 128: res5 at 2x2 when the
    network input is 64x64): the per-thread stores of rows moving above the
    clip start must stay inside their own clip.  Three clips, output buffer
    poisoned with NaN so a stray or missing store shows."""
    torch.manual_seed(13)
    n, t, cout, f = 3, 8, 64, 32
    h, w = hw
    cin = 8 * f
    dy = torch.randn(n, t, h, w, cout, device="cuda").bfloat16()
    wm = torch.randn(cout, 1, 1, cin, device="cuda") / 8
    wf, wd = conv.weights_to_bf16(wm)
    res = torch.randn(n, t, h, w, cin, device="cuda").bfloat16()
    g = dy.float() @ wf.float()
    adj = torch.zeros_like(g)
    adj[:, :-1, ..., :f] = g[:, 1:, ..., :f]
    adj[:, 1:, ..., f:2 * f] = g[:, :-1, ..., f:2 * f]
    adj[..., 2 * f:] = g[..., 2 * f:]
    ref_v = adj + res.float()
    out = torch.full((n, t, h, w, cin), float("nan"), device="cuda").bfloat16()
    dx = conv.conv_dgrad(dy, wd, (n, t, h, w, cin), fold=(f, f), residual=res, out=out)
    torch.cuda.synchronize()
    assert not torch.isnan(dx.float()).any()
    assert rel_err(dx, ref_v) < 1e-2
