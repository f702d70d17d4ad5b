"""GPU numerics of the tcgen05 conv engine against a plain fp32 torch
reference of the same op on the same bf16-rounded inputs."""
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
    (1, 4, 6, 6, 64, 64, 8),       # F=8 -> KC=8 slabs, no swizzle
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


def test_conv1x1_residual_relu():
    torch.manual_seed(1)
    dev = torch.device("cuda")
    x = torch.randn(2, 4, 8, 8, 64, device=dev).bfloat16()
    wt = (torch.randn(256, 64, device=dev) / 8).bfloat16()
    b = torch.randn(256, device=dev) * 0.1
    r = torch.randn(2, 4, 8, 8, 256, device=dev).bfloat16()
    y = conv.conv1x1_fwd(x, wt, b, relu=True, residual=r)
    ref = (x.float() @ wt.float().t() + b + r.float()).clamp_min(0)
    assert rel_err(y, ref) < 1e-2
