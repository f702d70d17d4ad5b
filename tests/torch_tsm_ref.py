"""TEST-ONLY plain PyTorch fp32 statement of TSM-ResNet-50 (build_tsm8f,
arch.cpp:140-161; run_unit net.cpp:85-126; loss net.cpp:141-146) used as the
numerics reference for the B200 network, with autograd for the gradients.
Parameters come from the GEMM-layout flat vector of ``TSMNet``."""
import torch
import torch.nn.functional as F


def unpack(net, vec):
    """flat GEMM-layout vector -> list of tensors in conv2d layout (co, ci, kh, kw)."""
    out = []
    for t in net.table:
        co, kh, kw, ci = t["dims"]
        x = vec[t["offset"]:t["offset"] + t["numel"]]
        if t["is_bias"]:
            out.append(x.reshape(co))
        else:
            out.append(x.reshape(co, kh, kw, ci)[..., :t["ci_ref"]].permute(0, 3, 1, 2))
    return out


def shift(x, n, t, fold):
    """kernels.cpp:97-125 on (N*T, C, H, W): [0,F) from t-1, [F,2F) from t+1."""
    nt, c, h, w = x.shape
    v = x.reshape(n, t, c, h, w)
    out = torch.zeros_like(v)
    out[:, 1:, :fold] = v[:, :-1, :fold]
    out[:, :-1, fold:2 * fold] = v[:, 1:, fold:2 * fold]
    out[:, :, 2 * fold:] = v[:, :, 2 * fold:]
    return out.reshape(nt, c, h, w)


def forward(params, x, shift_div=8):
    """x: [N][T][3][H][W] fp32 -> logits [N][classes]."""
    n, t = x.shape[:2]
    it = iter(params)
    h = x.reshape(n * t, *x.shape[2:])
    w, b = next(it), next(it)
    h = F.conv2d(h, w, b, stride=2, padding=3)           # conv1, linear
    h = F.max_pool2d(h, 3, 2, 1)                          # pool1
    cin = 64
    for s, (blocks, cout) in enumerate(zip((3, 4, 6, 3), (256, 512, 1024, 2048))):
        for bi in range(blocks):
            stride = 2 if (s > 0 and bi == 0) else 1
            w1, b1, w2, b2, w3, b3 = [next(it) for _ in range(6)]
            has_proj = stride != 1 or cin != cout
            xs = shift(h, n, t, cin // shift_div) if shift_div else h
            r = F.relu(F.conv2d(xs, w1, b1))
            r = F.relu(F.conv2d(r, w2, b2, stride=stride, padding=1))
            r = F.conv2d(r, w3, b3)
            if has_proj:
                wp, bp = next(it), next(it)
                skip = F.conv2d(h, wp, bp, stride=stride)
            else:
                skip = h
            h = F.relu(r + skip)
            cin = cout
    feat = h.reshape(n, t, *h.shape[1:]).mean(dim=(1, 3, 4))
    wf, bf = next(it), next(it)
    return F.linear(feat, wf.reshape(wf.shape[0], -1), bf)
