"""Guard bands around every output and workspace of the hot-path kernels.

compute-sanitizer is closed on this GPU pool (runs under it have left GPUs
needing a reset), so out-of-bounds writes are checked the direct way: each
output / workspace is a view into a larger buffer whose head and tail (64 KiB
each) hold a sentinel bit pattern, and after the launch both bands must be
bitwise unchanged.  Shapes are chosen for the edge cases of the tile and
store logic: partial tiles, clips shorter than one tile (per-thread stores
of shifted rows), strided scatter, sub-pixel dgrad classes, split-K
workspaces, CTA-pair kernels, the virtual-channel weight gradient, and the
1-D TMA bulk shift chain."""
import ctypes as C

import pytest
import torch

pytestmark = pytest.mark.gpu

from paper_1910_00932_b200 import _lib, conv  # noqa: E402
from paper_1910_00932_b200.shift import ShiftConfig, temporal_shift, temporal_shift_adjoint  # noqa: E402

GUARD = 64 * 1024  # bytes per band


class Guarded:
    """A tensor view with sentinel bands on both sides."""

    def __init__(self, shape, dtype, fill=None):
        esz = torch.empty(0, dtype=dtype).element_size()
        self.g = GUARD // esz
        n = 1
        for s in shape:
            n *= s
        self.buf = torch.empty(n + 2 * self.g, device="cuda", dtype=dtype)
        bits = self.buf.view(torch.uint8)
        bits.copy_(torch.randint(0, 256, bits.shape, device="cuda", dtype=torch.uint8))
        self.view = self.buf[self.g:self.g + n].view(shape)
        if fill is not None:
            self.view.copy_(fill)
        self.head = self.buf[:self.g].view(torch.uint8).clone()
        self.tail = self.buf[self.g + n:].view(torch.uint8).clone()

    def check(self):
        torch.cuda.synchronize()
        n = self.view.numel()
        assert torch.equal(self.buf[:self.g].view(torch.uint8), self.head), "write below the buffer"
        assert torch.equal(self.buf[self.g + n:].view(torch.uint8), self.tail), "write past the buffer"


def bf(*shape):
    return torch.randn(*shape, device="cuda").bfloat16()


FWD = [
    # n, t, h, w, cin, cout, k, stride, fold
    (2, 8, 6, 6, 256, 64, 1, 1, 32),      # fused shift, 32-channel slabs, partial last tile
    (3, 8, 2, 2, 256, 64, 1, 1, 32),      # clip shorter than a tile
    (2, 8, 5, 5, 64, 64, 1, 1, 8),        # 8-channel groups: three-frame tile kernel
    (1, 3, 17, 9, 64, 64, 1, 1, 8),       # ... partial tiles
    (1, 8, 14, 14, 1024, 256, 1, 1, 128),  # CTA pair
    (2, 4, 9, 7, 64, 64, 3, 1, 0),        # halo 3x3 (CTA pairs)
    (1, 3, 9, 7, 64, 64, 3, 1, 0),        # ... odd tile count
    (1, 4, 9, 7, 256, 256, 3, 1, 0),      # tcgen05 im2col 3x3
    (2, 4, 9, 7, 128, 128, 3, 1, 0),      # halo 3x3, 128 channels, streamed weights
    (1, 3, 9, 7, 128, 128, 3, 1, 0),      # ... odd tile count: padding tile in the last pair
    (2, 4, 9, 7, 128, 128, 3, 2, 0),      # strided 3x3, odd extent
    (2, 4, 9, 7, 128, 256, 1, 2, 0),      # strided projection
]


@pytest.mark.parametrize("case", FWD, ids=lambda c: "x".join(map(str, c)))
def test_conv_fwd_guards(case):
    n, t, h, w, cin, cout, k, s, f = case
    torch.manual_seed(1)
    x = bf(n, t, h, w, cin)
    wt = torch.randn(cout, k, k, cin, device="cuda").bfloat16() * (k * k * cin) ** -0.5
    ho, wo = conv.out_hw(h, w, k, s)
    y = Guarded((n, t, ho, wo, cout), torch.bfloat16)
    res = bf(n, t, ho, wo, cout) if s == 1 and k == 1 else None
    conv.conv_fwd(x, wt, torch.zeros(cout, device="cuda"), k=k, stride=s, fold=(f, f), relu=True,
                  residual=res, out=y.view)
    y.check()
    assert torch.isfinite(y.view.float()).all()


DGRAD = [
    (2, 8, 6, 6, 256, 64, 1, 1, 32, True),   # adjoint shift + skip (TMA epilogue)
    (3, 8, 2, 2, 256, 64, 1, 1, 32, True),   # short clips: per-thread shifted-row stores
    (2, 8, 5, 5, 64, 64, 1, 1, 8, True),     # narrow split, 64 channels: three-frame tiles
    (1, 3, 17, 9, 64, 64, 1, 1, 8, True),    # ... partial tiles
    (2, 4, 10, 8, 128, 256, 1, 2, 0, False),  # strided 1x1 scatter
    (2, 4, 10, 8, 128, 128, 3, 2, 0, False),  # sub-pixel 3x3 classes
    (2, 4, 9, 7, 64, 64, 3, 1, 0, False),     # halo dgrad
    (1, 3, 9, 7, 64, 64, 3, 1, 0, False),     # ... odd tile count
    (2, 4, 9, 7, 128, 128, 3, 1, 0, False),   # halo dgrad, 128 channels
    (1, 3, 9, 7, 128, 128, 3, 1, 0, False),   # ... odd tile count
]


@pytest.mark.parametrize("case", DGRAD, ids=lambda c: "x".join(map(str, c[:9])))
def test_conv_dgrad_guards(case):
    n, t, h, w, cin, cout, k, s, f, with_res = case
    torch.manual_seed(2)
    ho, wo = conv.out_hw(h, w, k, s)
    dy = bf(n, t, ho, wo, cout)
    _, wd = conv.weights_to_bf16(torch.randn(cout, k, k, cin, device="cuda") * 0.05)
    dx = Guarded((n, t, h, w, cin), torch.bfloat16)
    res = bf(n, t, h, w, cin) if with_res else None
    conv.conv_dgrad(dy, wd, (n, t, h, w, cin), k=k, stride=s, fold=(f, f), residual=res,
                    out=dx.view)
    dx.check()
    assert torch.isfinite(dx.view.float()).all()


WGRAD = [
    (2, 8, 6, 6, 256, 64, 1, 1, 32),      # swapped (c_out 64), shifted x, split-K
    (2, 8, 5, 5, 64, 64, 1, 1, 8),        # virtual channels
    (2, 8, 3, 3, 128, 64, 1, 1, 16),      # virtual channels, two M tiles, short clips
    (1, 8, 14, 14, 256, 256, 3, 1, 0),    # CTA pair im2col
    (1, 8, 14, 14, 1024, 256, 1, 1, 128),  # CTA pair, shifted x
    (2, 4, 9, 7, 64, 64, 3, 1, 0),        # halo wgrad
    (1, 3, 9, 7, 128, 128, 3, 1, 0),      # 3x3 128 channels (halo window kernel when enabled)
    (2, 4, 10, 8, 128, 128, 3, 2, 0),     # strided 3x3
]


@pytest.mark.parametrize("case", WGRAD, ids=lambda c: "x".join(map(str, c)))
def test_conv_wgrad_guards(case):
    n, t, h, w, cin, cout, k, s, f = case
    torch.manual_seed(3)
    x = bf(n, t, h, w, cin)
    ho, wo = conv.out_hw(h, w, k, s)
    dy = bf(n, t, ho, wo, cout)
    dw = Guarded((cout, k, k, cin), torch.float32)
    db = Guarded((cout,), torch.float32)
    nb = _lib.lib.tsm_conv_wgrad_workspace_bytes(n, t, h, w, cin, cout, k, s)
    ws = Guarded((max(nb, 16) // 4,), torch.float32)
    st = torch.cuda.current_stream().cuda_stream
    p = lambda g: C.c_void_p(g.view.data_ptr())  # noqa: E731
    _lib.check(_lib.lib.tsm_conv_wgrad(C.c_void_p(x.data_ptr()), C.c_void_p(dy.data_ptr()), p(dw),
                                       p(db), p(ws), n, t, h, w, cin, cout, k, s, f, f, st))
    for g in (dw, db, ws):
        g.check()
    ref = conv.conv_wgrad(x, dy, k=k, stride=s, fold=(f, f))
    assert torch.equal(dw.view, ref)  # same result with a fresh workspace


@pytest.mark.parametrize("shape,dtype", [((2, 8, 256, 28, 28), torch.float32),
                                         ((1, 8, 64, 7, 7), torch.bfloat16),
                                         ((2, 3, 24, 5, 3), torch.float16),
                                         ((1, 2, 8, 1, 1), torch.float64)])
def test_shift_guards(shape, dtype):
    x = torch.randn(*shape, device="cuda").to(dtype)
    for fn in (temporal_shift, temporal_shift_adjoint):
        y = Guarded(shape, dtype)
        fn(x, ShiftConfig(), out=y.view)
        y.check()
