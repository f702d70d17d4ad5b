"""GPU parity of the TSM-ResNet-50 training step.

* against a plain PyTorch fp32 statement of the same network (tests/
  torch_tsm_ref.py, autograd for gradients) on the same weights and input:
  logits, loss and every parameter gradient, relative L2 per tensor;
* against the reference itself (oracle/_ref: vidperf::Network over
  build_tsm8f(), weights from seed 42, input seed 43, as in
  gradcheck_test.cpp:10-11): forward logits at one clip.

* against the reference itself: every parameter gradient of
  Network::loss_gradients (net.cpp:160-272) for TSM-R50 on the tcgen05 path,
  at 2 clips of 64x64 (the sized build_tsm8f of ref_capi.cpp) and, marked
  slow, 1 clip of 224x224.

Tolerances (bf16 operands/activations, fp32 accumulation, 50 layers without
batch norm): logits rel-L2 <= 5e-2; loss within 1e-2; gradients
rel-L2 <= 5e-2 per tensor — except conv1.w and the input gradient, which are
intrinsically sensitive to bf16 operands: tests/bf16_sensitivity.py runs the
reference algorithm in fp64 with only the weights and the input rounded to
bf16 and already moves conv1.w by 12% and dL/dx by 22% at 2x64x64 (max-pool
argmax and ReLU decisions near ties flip); with the B200 path's storage
precision emulated the same script gives conv1.w 14.4% and dL/dx 26.4%, what
the GPU measures (profiles/r02/bf16_sensitivity_64.txt).  Those two get
bounds of 2e-1 / 3.5e-1 (64x64) and 1e-1 / 3.5e-1 (224x224).  Measured
values are printed."""
import numpy as np
import pytest
import torch

from paper_1910_00932_b200.network import TSMNet

import torch_tsm_ref as tref

pytestmark = pytest.mark.gpu


def rel_l2(a, b):
    a = a.double()
    b = b.double()
    return float((a - b).norm() / b.norm().clamp_min(1e-30))


def test_train_step_vs_torch_fp32(cuda):
    torch.manual_seed(0)
    net = TSMNet(batch=2).init_random(seed=1)
    x = torch.randn(2, 8, 3, 224, 224, device=cuda)
    # bf16-round the input and the weights so both sides see the same values
    x = x.bfloat16().float()
    with torch.no_grad():
        net.params.copy_(net.params.bfloat16().float())
    params = [p.clone().requires_grad_(True) for p in tref.unpack(net, net.params.clone())]
    logits_ref = tref.forward(params, x)
    loss_ref = (logits_ref ** 2).sum()
    loss_ref.backward()

    loss = net.train_step(x, update=False)
    torch.cuda.synchronize()
    logits = net.logits.clone()
    grads = tref.unpack(net, net.grads.clone())
    e_logit = rel_l2(logits, logits_ref)
    e_loss = abs(float(loss) - float(loss_ref)) / float(loss_ref)
    errs = {t["name"]: rel_l2(g, p.grad) for t, g, p in zip(net.table, grads, params)}
    worst = max(errs, key=errs.get)
    print(f"logits rel-L2 {e_logit:.3e}  loss rel {e_loss:.3e}  worst grad {worst} "
          f"{errs[worst]:.3e}  median grad {np.median(list(errs.values())):.3e}")
    assert e_logit <= 5e-2
    assert e_loss <= 1e-2
    assert errs[worst] <= 5e-2, errs


@pytest.mark.parametrize("hw", [64, 63])
def test_input_grad_vs_torch(cuda, hw):
    """dL/dx (the stem conv's input gradient, tsm_net_input_grad) against
    torch autograd on the same bf16-rounded weights and input; also the
    stem-output gradient's effect on conv1.w.  Printed: the errors."""
    torch.manual_seed(5)
    net = TSMNet(batch=2, height=hw, width=hw).init_random(seed=3)
    x = torch.randn(2, 8, 3, hw, hw, device=cuda).bfloat16().float()
    with torch.no_grad():
        net.params.copy_(net.params.bfloat16().float())
    params = [p.clone().requires_grad_(True) for p in tref.unpack(net, net.params.clone())]
    xr = x.clone().requires_grad_(True)
    (tref.forward(params, xr) ** 2).sum().backward()
    net.train_step(x, update=False)
    gx = net.input_grad()
    torch.cuda.synchronize()
    e_in = rel_l2(gx, xr.grad)
    grads = tref.unpack(net, net.grads.clone())
    e_w = rel_l2(grads[0], params[0].grad)
    print(f"{hw}x{hw}: input grad rel-L2 {e_in:.3e}; conv1.w {e_w:.3e}")
    # (torch's own conv2d runs TF32 on the GPU by default: both sides carry
    # operand rounding; bound as against the reference)
    assert e_in <= INPUT_GRAD_TOL


@pytest.mark.parametrize("hw", [63, 64])
def test_train_step_small_extents_vs_torch(cuda, hw):
    # odd extents take the materialised-im2col stem, even ones the
    # space-to-depth stem: both against the same torch fp32 statement
    torch.manual_seed(5)
    net = TSMNet(batch=1, height=hw, width=hw).init_random(seed=3)
    x = torch.randn(1, 8, 3, hw, hw, device=cuda).bfloat16().float()
    with torch.no_grad():
        net.params.copy_(net.params.bfloat16().float())
    params = [p.clone().requires_grad_(True) for p in tref.unpack(net, net.params.clone())]
    logits_ref = tref.forward(params, x)
    (logits_ref ** 2).sum().backward()
    net.train_step(x, update=False)
    torch.cuda.synchronize()
    e_logit = rel_l2(net.logits.clone(), logits_ref)
    grads = tref.unpack(net, net.grads.clone())
    errs = {t["name"]: rel_l2(g, p.grad) for t, g, p in zip(net.table, grads, params)}
    print(f"{hw}x{hw}: logits rel-L2 {e_logit:.3e} conv1.w {errs['conv1.w']:.3e} "
          f"conv1.b {errs['conv1.b']:.3e}")
    assert e_logit <= 5e-2
    # conv1.w sums over few pixels at these extents: bf16 rounding of the
    # incoming gradient is not averaged out (measured 0.12 for BOTH stem
    # paths, vs 0.03 at 224x224)
    assert errs["conv1.w"] <= 2e-1 and errs["conv1.b"] <= 1e-1


def test_forward_vs_reference_network(cuda, ref):
    # vidperf::Network(build_tsm8f(), 42) on random_normal(input_shape, 43)
    rnet = ref.net("tsm8f", (1, 8), 42)
    flat = rnet.param_vector()
    x = ref.random_normal((1, 8, 3, 224, 224), 43)
    y_ref = rnet.forward(x).reshape(1, 400)
    net = TSMNet(batch=1).load_reference(flat)
    y = net.forward(torch.from_numpy(x).to(cuda))
    torch.cuda.synchronize()
    e = rel_l2(y.cpu(), torch.from_numpy(y_ref))
    loss_ref = float((y_ref ** 2).sum())
    print(f"reference logits rel-L2 {e:.3e}; loss ref {loss_ref:.4e} gpu {float((y ** 2).sum()):.4e}")
    assert abs(loss_ref - 4.836e8) / 4.836e8 < 1e-3   # SURVEY §0 trap 7
    assert e <= 5e-2


def ref_tensor_errors(net, g, g_ref):
    """Per-tensor rel-L2 of two gradient vectors in the reference's flat order
    and layout (net.cpp:250-270)."""
    pos, errs = 0, {}
    for t in net.table:
        co, kh, kw, _ = t["dims"]
        n = co * kh * kw * t["ci_ref"]
        errs[t["name"]] = rel_l2(torch.from_numpy(g[pos:pos + n]),
                                 torch.from_numpy(g_ref[pos:pos + n]))
        pos += n
    assert pos == g_ref.size
    return errs


# conv1.w bound per extent (see the module docstring)
CONV1_W_TOL = {64: 2e-1, 224: 1e-1}
INPUT_GRAD_TOL = 3.5e-1


def _grads_vs_reference(cuda, ref, n, hw):
    # vidperf::Network(build_tsm8f() at hw x hw, seed 42) on random_normal
    # input seed 43, as gradcheck_test.cpp:10-11 seeds it; the same weights
    # (fp64 -> fp32 masters) and input on the GPU.  TSM-R50's blocks all run
    # on the tcgen05 kernels (the fused shift + 1x1 conv included).
    rnet = ref.net_sized(hw, hw, 42)
    flat = rnet.param_vector()
    x = ref.random_normal((n, 8, 3, hw, hw), 43)
    loss_ref, g_ref, gx_ref = rnet.loss_gradients(x)
    net = TSMNet(batch=n, height=hw, width=hw).load_reference(flat)
    loss = float(net.train_step(torch.from_numpy(x).to(cuda), update=False))
    gx = net.input_grad(torch.float64).cpu()
    torch.cuda.synchronize()
    errs = ref_tensor_errors(net, net.grads_reference(), g_ref)
    e_in = rel_l2(gx, torch.from_numpy(gx_ref))
    conv1_w = errs.pop("conv1.w")
    worst = max(errs, key=errs.get)
    e_loss = abs(loss - loss_ref) / abs(loss_ref)
    print(f"TSM-R50 {n}x{hw}x{hw} vs reference loss_gradients: loss {loss:.6e} ref "
          f"{loss_ref:.6e} (rel {e_loss:.2e}); grads rel-L2 median "
          f"{np.median(list(errs.values())):.2e}, worst (without conv1.w) {worst} "
          f"{errs[worst]:.2e}; conv1.w {conv1_w:.2e}; input gradient {e_in:.2e}")
    print("  " + " ".join(f"{k}={v:.1e}" for k, v in errs.items()))
    assert e_loss <= 1e-2
    assert errs[worst] <= 5e-2, errs
    assert conv1_w <= CONV1_W_TOL[hw]
    assert e_in <= INPUT_GRAD_TOL


def test_loss_gradients_vs_reference_network_64(cuda, ref):
    # 2 clips: also the multi-clip path of the small-extent tiles (res5 is
    # 2x2 here, shorter than one 128-row tile per clip)
    _grads_vs_reference(cuda, ref, 2, 64)


@pytest.mark.slow
def test_loss_gradients_vs_reference_network_224(cuda, ref):
    _grads_vs_reference(cuda, ref, 1, 224)


@pytest.mark.parametrize("shift", [(1, 8), (0, 1)])
def test_micro_tsm_vs_reference(cuda, ref, shift):
    # build_micro_tsm (arch.cpp:220-233): input (1,4,8,5,5), two 16-channel
    # units (width 4 -> the direct-conv block path), 4 classes; weights from
    # seed 42 and input seed 43 as in gradcheck_test.cpp:8-21.  Logits, loss
    # and every parameter gradient against the reference's own
    # Network::loss_gradients (fp64) — bf16 activations here.
    from paper_1910_00932_b200.shift import Rational, ShiftConfig
    rnet = ref.net("micro-tsm", shift, 42)
    flat = rnet.param_vector()
    x = ref.random_normal((1, 4, 8, 5, 5), 43)
    y_ref = rnet.forward(x).reshape(1, 4)
    loss_ref, g_ref, _ = rnet.loss_gradients(x)
    cfg = ShiftConfig.symmetric(Rational(*shift)) if shift[0] else None
    net = TSMNet(batch=1, frames=4, height=5, width=5, classes=4, shift=cfg,
                 arch="micro-tsm").load_reference(flat)
    assert net.reference_param_count() == rnet.param_count() == 772
    loss = float(net.train_step(torch.from_numpy(x).to(cuda), update=False))
    torch.cuda.synchronize()
    e_logit = rel_l2(net.logits.cpu(), torch.from_numpy(y_ref))
    errs = ref_tensor_errors(net, net.to_reference(net.grads), g_ref)
    worst = max(errs, key=errs.get)
    print(f"micro-tsm shift {shift}: logits rel-L2 {e_logit:.3e} loss {loss:.6e} ref "
          f"{loss_ref:.6e} worst grad {worst} {errs[worst]:.3e}")
    assert e_logit <= 2e-2
    assert abs(loss - loss_ref) / abs(loss_ref) <= 4e-2
    # bf16 activations at 5x5: rounding is not averaged out (measured worst
    # ~5.6e-2, res2.0.w1); same bound as the full network
    assert errs[worst] <= 1e-1, errs


def test_param_count_matches_reference(cuda):
    net = TSMNet(batch=1)
    assert net.reference_param_count() == 24301072   # cost_test.cpp:72
    assert len(net.table) == 108                      # 53 convs + fc, w and b each


_SUB = r"""
import sys, torch
sys.path.insert(0, {root!r})
from paper_1910_00932_b200.network import TSMNet
torch.manual_seed(0)
net = TSMNet(batch=2).init_random(seed=1)
x = torch.randn(2, 8, 3, 224, 224, device="cuda")
loss = net.train_step(x, update=False)
torch.cuda.synchronize()
torch.save({{"loss": float(loss), "grads": net.grads.cpu(), "logits": net.logits.cpu()}}, {out!r})
"""


def _run_step(tmp_path, name, env):
    import os
    import subprocess
    import sys
    from pathlib import Path
    out = tmp_path / f"{name}.pt"
    root = str(Path(__file__).resolve().parents[1])
    r = subprocess.run([sys.executable, "-c", _SUB.format(root=root, out=str(out))],
                       env={**os.environ, **env}, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    return torch.load(out)


def test_train_step_deterministic_and_stream_independent(cuda, tmp_path):
    # bitwise run-to-run determinism of the whole step (no float atomics,
    # fixed-order reductions), and the side-stream weight gradients give the
    # same bits as the serialised step (TSM_SIDE_STREAM=0)
    a = _run_step(tmp_path, "a", {})
    b = _run_step(tmp_path, "b", {})
    c = _run_step(tmp_path, "c", {"TSM_SIDE_STREAM": "0"})
    assert torch.equal(a["grads"], b["grads"]) and a["loss"] == b["loss"]
    assert torch.equal(a["grads"], c["grads"]) and torch.equal(a["logits"], c["logits"])


def test_residual_through_mma_matches_epilogue_residual(cuda, tmp_path):
    # TSM_FUSE_RES=0 adds the residuals in the epilogue instead of as identity
    # k-blocks: same math, fp32 summation order differs -> tolerance
    a = _run_step(tmp_path, "fused", {})
    b = _run_step(tmp_path, "epi", {"TSM_FUSE_RES": "0"})
    e_logit = rel_l2(a["logits"], b["logits"])
    e_grad = rel_l2(a["grads"], b["grads"])
    print(f"fused vs epilogue residual: logits {e_logit:.2e} grads {e_grad:.2e}")
    assert e_logit < 1e-2 and e_grad < 2e-2


@pytest.mark.gpu
def test_in_step_shift_conv1_probe(cuda):
    """bench.py's in-step roofline probe: the res2 units with 256 input
    channels (res2.1, res2.2) each launch one fused shift + conv1 per step;
    nothing is recorded once the probe is stopped."""
    from paper_1910_00932_b200 import _lib
    net = TSMNet(batch=1, height=64, width=64).init_random(seed=5)
    x = torch.randn(1, 8, 3, 64, 64, device=cuda)
    net.train_step(x, update=False)
    _lib.probe_shift_conv1(256, 64)
    for _ in range(2):
        net.train_step(x, update=False)
    _lib.probe_shift_conv1(0)
    n, us, px = _lib.probe_shift_conv1_read()
    assert n == 4 and us > 0 and px == 1 * 8 * 16 * 16
    net.train_step(x, update=False)
    assert _lib.probe_shift_conv1_read()[0] == 4


def test_graph_replay_matches_eager(cuda):
    """tsm_net_set_graph: the captured step replayed three times (with the
    SGD update, new hyperparameters each step) gives the eager step's bits:
    loss, gradients and updated parameters."""
    from paper_1910_00932_b200 import _lib
    x = torch.randn(2, 8, 3, 64, 64, device=cuda)
    a = TSMNet(batch=2, height=64, width=64).init_random(seed=9)
    b = TSMNet(batch=2, height=64, width=64).init_random(seed=9).set_graph(True)
    for i in range(3):
        kw = dict(lr=1e-12 * (i + 1), momentum=0.9, weight_decay=1e-4)
        la = float(a.train_step(x, **kw))
        l0 = _lib.launch_count()
        lb = float(b.train_step(x, **kw))
        launches = _lib.launch_count() - l0
        torch.cuda.synchronize()
        assert la == lb, (i, la, lb)
        assert torch.equal(a.grads, b.grads) and torch.equal(a.params, b.params), i
        assert launches > 100   # the replay is counted as the kernels it runs


_STEP_DIGEST = r"""
import hashlib, sys, torch
sys.path.insert(0, {root!r})
from paper_1910_00932_b200.network import TSMNet
net = TSMNet(batch=2, height={hw}, width={hw}).init_random(seed=5)
x = torch.randn(2, 8, 3, {hw}, {hw}, generator=torch.Generator().manual_seed(7)).cuda()
y = net.forward(x)
loss = net.train_step(x, update=False)
torch.cuda.synchronize()
h = hashlib.sha256()
h.update(y.detach().float().cpu().numpy().tobytes())
h.update(net.grads.detach().cpu().numpy().tobytes())
print(h.hexdigest())
"""


@pytest.mark.gpu
@pytest.mark.parametrize("hw", [64, 224])
@pytest.mark.parametrize("switch", ["TSM_STEM_POOL", "TSM_STEM_POOL_BWD"])
def test_fused_stem_pool_bitwise_equals_two_kernels(hw, switch):
    """The fused stem conv + max pool forward (TSM_STEM_POOL) and the pool
    backward fused into the stem weight gradient (TSM_STEM_POOL_BWD), both on
    by default, give bitwise the logits and every gradient of the separate
    kernels: two processes, one per path."""
    import os
    import subprocess
    import sys
    from pathlib import Path
    code = _STEP_DIGEST.format(root=str(Path(__file__).resolve().parents[1]), hw=hw)
    digests = []
    for v in ("1", "0"):
        r = subprocess.run([sys.executable, "-c", code], env=dict(os.environ, **{switch: v}),
                           capture_output=True, text=True, timeout=900)
        assert r.returncode == 0, r.stderr[-3000:]
        digests.append(r.stdout.strip().splitlines()[-1])
    assert digests[0] == digests[1]
