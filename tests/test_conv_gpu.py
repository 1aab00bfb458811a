"""The library's fp32 3x3 convolutions (csrc/conv_f32.cu via conv.py)
against an fp64 reference of the same op (cuDNN in fp64), at the CIFAR
ResNet-20 shapes: forward, data gradient, weight gradient, the autograd
function with partial backprop, graph capture, and the cuDNN routing for
shapes without a kernel."""

from __future__ import annotations

import pytest
import torch
import torch.nn.functional as F

pytestmark = pytest.mark.gpu

CL = torch.channels_last
SHAPES = [(16, 32), (32, 16), (64, 8)]
# fp32 FFMA with a different summation order than the fp64 reference:
# max |err| / max |ref| (cuDNN's own fp32 algorithms land at ~5e-7)
TOL = 1e-5


def _rel(a, ref):
    return float((a.double() - ref).abs().max() / ref.abs().max())


def _data(c, hw, n, seed=0):
    g = torch.Generator(device="cuda").manual_seed(seed)
    x = torch.randn(n, c, hw, hw, device="cuda", generator=g).to(memory_format=CL)
    w = (torch.randn(c, c, 3, 3, device="cuda", generator=g) / (3 * c ** 0.5)).to(memory_format=CL)
    gy = torch.randn(n, c, hw, hw, device="cuda", generator=g).to(memory_format=CL)
    return x, w, gy


def _ref(x, w, gy):
    xd, wd, gyd = x.double(), w.double(), gy.double()
    y = F.conv2d(xd, wd, padding=1)
    gx, gw, _ = torch.ops.aten.convolution_backward(gyd, xd, wd, None, (1, 1), (1, 1), (1, 1), False, (0, 0), 1,
                                                    (True, True, False))
    return y, gx, gw


@pytest.mark.parametrize("c,hw", SHAPES)
@pytest.mark.parametrize("n", [1, 3, 128])
def test_conv_kernels_match_fp64(c, hw, n):
    from paper_2203_06638_b200 import conv

    x, w, gy = _data(c, hw, n)
    y_ref, gx_ref, gw_ref = _ref(x, w, gy)
    y = conv.conv_fwd(x, w)
    gx = conv.conv_fwd(gy, w, dgrad=True)
    gw = conv.conv_wgrad(x, gy, w)
    assert y.is_contiguous(memory_format=CL) and gw.is_contiguous(memory_format=CL)
    assert _rel(y, y_ref) < TOL
    assert _rel(gx, gx_ref) < TOL
    assert _rel(gw, gw_ref) < TOL


@pytest.mark.parametrize("c,hw", SHAPES)
def test_conv_wgrad_deterministic(c, hw):
    from paper_2203_06638_b200 import conv

    x, w, gy = _data(c, hw, 64, seed=1)
    a = conv.conv_wgrad(x, gy, w)
    b = conv.conv_wgrad(x, gy, w)
    assert torch.equal(a, b)


def test_conv_zero_padding_edges():
    """A constant image: border outputs see fewer taps (zero padding)."""
    from paper_2203_06638_b200 import conv

    c, hw = 16, 32
    x = torch.ones(2, c, hw, hw, device="cuda").to(memory_format=CL)
    w = torch.ones(c, c, 3, 3, device="cuda").to(memory_format=CL)
    y = conv.conv_fwd(x, w)
    assert float(y[0, 0, 0, 0]) == 4 * c and float(y[0, 0, 5, 5]) == 9 * c and float(y[1, 3, 0, 7]) == 6 * c


@pytest.mark.parametrize("which", ["both", "input", "weight"])
def test_conv3x3_module_autograd(which):
    from paper_2203_06638_b200.conv import Conv3x3

    torch.manual_seed(0)
    m = Conv3x3(32, 32, 1).cuda().to(memory_format=CL)
    x, _, gy = _data(32, 16, 8, seed=2)
    x.requires_grad_(which in ("both", "input"))
    m.weight.requires_grad_(which in ("both", "weight"))
    y = m(x)
    y.backward(gy)
    xd = x.detach().double().requires_grad_(x.requires_grad)
    wd = m.weight.detach().double().requires_grad_(m.weight.requires_grad)
    yd = F.conv2d(xd, wd, padding=1)
    yd.backward(gy.double())
    assert _rel(y.detach(), yd.detach()) < TOL
    if which in ("both", "input"):
        assert _rel(x.grad, xd.grad) < TOL
    else:
        assert x.grad is None
    if which in ("both", "weight"):
        assert _rel(m.weight.grad, wd.grad) < TOL
    else:
        assert m.weight.grad is None


def test_conv3x3_routes_other_cases_to_cudnn(monkeypatch):
    """No kernel for the shape / dtype, autocast, or LPP_CONV=cudnn: F.conv2d
    (no library launch); the supported shapes launch ours."""
    from paper_2203_06638_b200 import _native as N
    from paper_2203_06638_b200.conv import Conv3x3

    def launches(fn):
        torch.cuda.synchronize()
        l0 = N.launch_count()
        out = fn()
        torch.cuda.synchronize()
        return out, N.launch_count() - l0

    x16 = torch.randn(2, 16, 16, 16, device="cuda").to(memory_format=CL)   # (16, 16): no kernel
    m = Conv3x3(16, 16, 1).cuda().to(memory_format=CL)
    y, k = launches(lambda: m(x16))
    assert k == 0 and torch.allclose(y, F.conv2d(x16, m.weight, padding=1), atol=1e-5)
    x32 = torch.randn(2, 16, 32, 32, device="cuda").to(memory_format=CL)
    with torch.autocast("cuda", dtype=torch.bfloat16):
        assert launches(lambda: m(x32))[1] == 0
    assert launches(lambda: m(x32.double()) if False else m(x32))[1] == 1
    assert launches(lambda: Conv3x3(16, 32, 2).cuda().to(memory_format=CL)(x32))[1] == 1   # stride-2 kernel
    monkeypatch.setenv("LPP_CONV", "cudnn")
    assert launches(lambda: m(x32))[1] == 0


def test_conv_in_cuda_graph():
    from paper_2203_06638_b200 import conv

    x, w, gy = _data(64, 8, 16, seed=3)
    y_ref, gx_ref, gw_ref = _ref(x, w, gy)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        conv.conv_fwd(x, w), conv.conv_fwd(gy, w, dgrad=True), conv.conv_wgrad(x, gy, w)
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        out = (conv.conv_fwd(x, w), conv.conv_fwd(gy, w, dgrad=True), conv.conv_wgrad(x, gy, w))
    for o in out:
        o.zero_()
    g.replay()
    torch.cuda.synchronize()
    assert _rel(out[0], y_ref) < TOL and _rel(out[1], gx_ref) < TOL and _rel(out[2], gw_ref) < TOL


def test_conv_rejects_unsupported_shape():
    from paper_2203_06638_b200 import _native as N
    from paper_2203_06638_b200 import conv

    x = torch.randn(2, 16, 16, 16, device="cuda").to(memory_format=CL)
    w = torch.randn(16, 16, 3, 3, device="cuda").to(memory_format=CL)
    with pytest.raises(ValueError, match="no kernel"):
        conv.conv_fwd(x, w)
    assert N.lib.lpp_conv3x3_wgrad_workspace(2, 16, 16) == 0


def test_wgrad_arrival_cells_reused_stay_zero():
    """One launch per weight gradient: the last cluster resets the arrival
    counters, so a set reused by stream-ordered calls gives the same bits."""
    from paper_2203_06638_b200 import conv

    for c, hw in SHAPES:
        x, w, gy = _data(c, hw, 32, seed=4)
        cells = conv.arrival_cells("cuda")
        outs = [conv.conv_wgrad(x, gy, w, cells) for _ in range(4)]
        assert all(torch.equal(outs[0], o) for o in outs[1:])
        assert int(cells.abs().sum()) == 0
        _, _, gw_ref = _ref(x, w, gy)
        assert _rel(outs[0], gw_ref) < TOL


def test_partial_backprop_skips_unneeded_kernels():
    """autograd.grad over a subset of weights (a PASSM+ block): layers above
    the block run dgrad only, the block's input-most layer no dgrad."""
    from paper_2203_06638_b200 import _native as N
    from paper_2203_06638_b200 import conv
    from paper_2203_06638_b200.conv import Conv3x3

    torch.manual_seed(1)
    seq = torch.nn.Sequential(Conv3x3(16, 16), torch.nn.ReLU(), Conv3x3(16, 16)).cuda().to(memory_format=CL)
    x = torch.randn(4, 16, 32, 32, device="cuda").to(memory_format=CL)
    c1, c2 = seq[0], seq[2]

    def grads(targets):
        conv.mark_weight_grads(seq, targets)
        y = seq(x)
        torch.cuda.synchronize()
        l0 = N.launch_count()
        g = torch.autograd.grad((y * y).sum(), targets)
        torch.cuda.synchronize()
        return g, N.launch_count() - l0

    (g2,), n2 = grads([c2.weight])
    assert n2 == 1                         # conv2 wgrad only
    (g1,), n1 = grads([c1.weight])
    assert n1 == 2                         # conv2 dgrad + conv1 wgrad
    (a1, a2), n12 = grads([c1.weight, c2.weight])
    assert n12 == 3
    xd = x.double()
    w1 = c1.weight.detach().double().requires_grad_()
    w2 = c2.weight.detach().double().requires_grad_()
    yd = F.conv2d(F.relu(F.conv2d(xd, w1, padding=1)), w2, padding=1)
    r1, r2 = torch.autograd.grad((yd * yd).sum(), [w1, w2])
    for got, ref in ((g1, r1), (g2, r2), (a1, r1), (a2, r2)):
        assert _rel(got, ref) < TOL
    conv.mark_weight_grads(seq, list(seq.parameters()))


SHAPES_1X1 = [(16, 32, 32), (32, 64, 16)]


@pytest.mark.parametrize("ci,co,hw", SHAPES_1X1)
@pytest.mark.parametrize("n", [1, 3, 128])
def test_conv1x1s2_kernels_match_fp64(ci, co, hw, n):
    """The projection shortcut (1x1, stride 2): forward, dX (zero at the
    odd pixels), dW — against fp64."""
    from paper_2203_06638_b200 import conv

    g = torch.Generator(device="cuda").manual_seed(5)
    x = torch.randn(n, ci, hw, hw, device="cuda", generator=g).to(memory_format=CL)
    w = (torch.randn(co, ci, 1, 1, device="cuda", generator=g) / ci ** 0.5).to(memory_format=CL)
    gy = torch.randn(n, co, hw // 2, hw // 2, device="cuda", generator=g).to(memory_format=CL)
    xd, wd, gyd = x.double(), w.double(), gy.double()
    y_ref = F.conv2d(xd, wd, stride=2)
    gx_ref, gw_ref, _ = torch.ops.aten.convolution_backward(gyd, xd, wd, None, (2, 2), (0, 0), (1, 1), False,
                                                            (0, 0), 1, (True, True, False))
    y = conv.conv1x1s2(x, w, 0)
    gx = conv.conv1x1s2(gy, w, 1)
    cells = conv.arrival_cells("cuda")
    gw = conv.conv1x1s2(x, w, 2, gy, cells)
    gw2 = conv.conv1x1s2(x, w, 2, gy, cells)
    assert y.shape == y_ref.shape and gx.shape == gx_ref.shape and gw.shape == gw_ref.shape
    assert _rel(y, y_ref) < TOL and _rel(gx, gx_ref) < TOL and _rel(gw, gw_ref) < TOL
    assert torch.equal(gw, gw2) and int(cells.abs().sum()) == 0
    assert float(gx[:, :, 1::2, :].abs().max()) == 0.0


def test_conv1x1_module_routes_and_grads():
    from paper_2203_06638_b200.conv import Conv1x1

    torch.manual_seed(2)
    m = Conv1x1(16, 32, 2).cuda().to(memory_format=CL)
    x = torch.randn(8, 16, 32, 32, device="cuda").to(memory_format=CL).requires_grad_()
    y = m(x)
    gy = torch.randn_like(y)
    y.backward(gy)
    xd = x.detach().double().requires_grad_()
    wd = m.weight.detach().double().requires_grad_()
    F.conv2d(xd, wd, stride=2).backward(gy.double())
    assert _rel(x.grad, xd.grad) < TOL and _rel(m.weight.grad, wd.grad) < TOL
    s1 = Conv1x1(16, 32, 1).cuda().to(memory_format=CL)      # stride 1: cuDNN
    x1 = torch.randn(2, 16, 8, 8, device="cuda").to(memory_format=CL)
    assert torch.allclose(s1(x1), F.conv2d(x1, s1.weight), atol=1e-5)


@pytest.mark.parametrize("ci,co,hw", SHAPES_1X1)
@pytest.mark.parametrize("n", [1, 3, 128])
def test_conv3x3s2_kernels_match_fp64(ci, co, hw, n):
    """The stage-opening 3x3 stride-2 convolution: forward, quad dgrad, wgrad."""
    from paper_2203_06638_b200 import conv

    g = torch.Generator(device="cuda").manual_seed(6)
    x = torch.randn(n, ci, hw, hw, device="cuda", generator=g).to(memory_format=CL)
    w = (torch.randn(co, ci, 3, 3, device="cuda", generator=g) / (3 * ci ** 0.5)).to(memory_format=CL)
    gy = torch.randn(n, co, hw // 2, hw // 2, device="cuda", generator=g).to(memory_format=CL)
    xd, wd, gyd = x.double(), w.double(), gy.double()
    y_ref = F.conv2d(xd, wd, stride=2, padding=1)
    gx_ref, gw_ref, _ = torch.ops.aten.convolution_backward(gyd, xd, wd, None, (2, 2), (1, 1), (1, 1), False,
                                                            (0, 0), 1, (True, True, False))
    cells = conv.arrival_cells("cuda")
    y = conv.conv3x3s2(x, w, 0)
    gx = conv.conv3x3s2(gy, w, 1)
    gw = conv.conv3x3s2(x, w, 2, gy, cells)
    assert y.shape == y_ref.shape and gx.shape == gx_ref.shape and gw.shape == gw_ref.shape
    assert _rel(y, y_ref) < TOL and _rel(gx, gx_ref) < TOL and _rel(gw, gw_ref) < TOL
    assert torch.equal(gw, conv.conv3x3s2(x, w, 2, gy, cells)) and int(cells.abs().sum()) == 0


def test_conv3x3_stride2_module_grads():
    from paper_2203_06638_b200.conv import Conv3x3

    torch.manual_seed(3)
    m = Conv3x3(32, 64, 2).cuda().to(memory_format=CL)
    x = torch.randn(8, 32, 16, 16, device="cuda").to(memory_format=CL).requires_grad_()
    y = m(x)
    gy = torch.randn_like(y)
    y.backward(gy)
    xd = x.detach().double().requires_grad_()
    wd = m.weight.detach().double().requires_grad_()
    yd = F.conv2d(xd, wd, stride=2, padding=1)
    yd.backward(gy.double())
    assert _rel(y.detach(), yd.detach()) < TOL
    assert _rel(x.grad, xd.grad) < TOL and _rel(m.weight.grad, wd.grad) < TOL


@pytest.mark.parametrize("cin,cout,stride,hw", [(16, 16, 1, 32), (16, 32, 2, 32), (32, 64, 2, 16), (64, 64, 1, 8)])
def test_basic_block_fused_bn_matches_fp64(cin, cout, stride, hw):
    """A ResNet basic block on the native path — convolutions with fused
    BatchNorm statistics, bn_act (BatchNorm + residual + ReLU in one pass) —
    against the same block in fp64 on torch's modules: output, running
    statistics, and every gradient."""
    import copy

    from paper_2203_06638_b200 import _native as N
    from paper_2203_06638_b200.objectives import _Basic

    torch.manual_seed(4)
    blk = _Basic(cin, cout, stride).cuda().to(memory_format=CL)
    for m in blk.modules():
        if isinstance(m, torch.nn.BatchNorm2d):
            m.weight.data.uniform_(0.5, 1.5)
            m.bias.data.uniform_(-0.5, 0.5)
    ref = copy.deepcopy(blk).double()
    x = torch.randn(16, cin, hw, hw, device="cuda").to(memory_format=CL).requires_grad_()
    xd = x.detach().double().requires_grad_()
    l0 = N.launch_count()
    y = blk(x)
    n_fwd = N.launch_count() - l0
    yd = ref(xd)
    gy = torch.randn_like(y)
    y.backward(gy)
    yd.backward(gy.double())
    tol = 2e-5
    assert _rel(y.detach(), yd.detach()) < tol
    assert _rel(x.grad, xd.grad) < tol
    for (name, p), (_, pd) in zip(blk.named_parameters(), ref.named_parameters()):
        assert _rel(p.grad, pd.grad) < tol, name
    for (name, b), (_, bd) in zip(blk.named_buffers(), ref.named_buffers()):
        if b.dtype.is_floating_point:
            assert _rel(b, bd) < tol, name
    # conv + BatchNorm pass per convolution: 2 x 2, plus 2 for the projection,
    # plus the tap-major weight copy of each stride-1 forward with C >= 32
    tapmajor = sum(1 for m in (blk.conv1, blk.conv2) if m.stride == (1, 1) and m.out_channels >= 32)
    assert n_fwd == (4 if blk.shortcut is None else 6) + tapmajor


@pytest.mark.parametrize("n", [1, 3, 128])
def test_stem_kernels_match_fp64(n):
    """The stem (3 -> 16 on the NCHW batch): forward, fused statistics, dW."""
    from paper_2203_06638_b200 import conv

    g = torch.Generator(device="cuda").manual_seed(7)
    x = torch.randn(n, 3, 32, 32, device="cuda", generator=g)                  # NCHW, as gathered
    w = (torch.randn(16, 3, 3, 3, device="cuda", generator=g) / 5).to(memory_format=CL)
    gy = torch.randn(n, 16, 32, 32, device="cuda", generator=g).to(memory_format=CL)
    xd, wd = x.double(), w.double()
    y_ref = F.conv2d(xd, wd, padding=1)
    _, gw_ref, _ = torch.ops.aten.convolution_backward(gy.double(), xd, wd, None, (1, 1), (1, 1), (1, 1), False,
                                                       (0, 0), 1, (False, True, False))
    cells = conv.arrival_cells("cuda", 2)
    y, sums = conv.stem(x, w, 0, stats=cells[8:])
    assert y.is_contiguous(memory_format=CL) and _rel(y, y_ref) < TOL
    ref_sums = torch.stack([y_ref.sum((0, 2, 3)), (y_ref * y_ref).sum((0, 2, 3))], 1).reshape(-1)
    assert _rel(sums, ref_sums) < TOL
    gw = conv.stem(x, None, 2, gy, cells)
    assert gw.shape == (16, 3, 3, 3) and _rel(gw, gw_ref) < TOL
    assert int(cells.abs().sum()) == 0


def test_resnet20_native_matches_fp64(monkeypatch):
    """The whole fp32 ResNet-20 on the native path (stem, 20 convolutions,
    fused BatchNorm / residual / ReLU) against an fp64 copy on torch's
    modules: logits, every parameter gradient, the running statistics —
    each within 3x the error torch's own fp32 path (cuDNN, TF32 off) makes
    against the same fp64 copy (20 BatchNorm layers amplify fp32 rounding),
    and never above 2e-3."""
    import copy

    from paper_2203_06638_b200 import _native as N
    from paper_2203_06638_b200.objectives import CifarResNet20

    torch.backends.cudnn.allow_tf32 = False
    torch.manual_seed(8)
    model = CifarResNet20().cuda().to(memory_format=CL)
    torch_fp32 = copy.deepcopy(model)
    ref = copy.deepcopy(model).double()
    x = torch.randn(64, 3, 32, 32, device="cuda")
    gy = torch.randn(64, 10, device="cuda")
    l0 = N.launch_count()
    y = model(x)
    # stem + 18 + 2 projections, one BatchNorm pass each, and the tap-major
    # weight copy of the 10 stride-1 forwards with C >= 32
    assert N.launch_count() - l0 == 21 + 21 + 10
    y.backward(gy)
    yd = ref(x.double())
    yd.backward(gy.double())
    monkeypatch.setenv("LPP_CONV", "cudnn")
    yt = torch_fp32(x.contiguous(memory_format=CL))
    yt.backward(gy)
    monkeypatch.delenv("LPP_CONV")

    def ok(ours, theirs, exact, what):
        e_ours, e_torch = _rel(ours, exact), _rel(theirs, exact)
        assert e_ours < max(1e-5, 3 * e_torch) and e_ours < 2e-3, (what, e_ours, e_torch)

    ok(y.detach(), yt.detach(), yd.detach(), "logits")
    for (name, p), (_, pt), (_, pd) in zip(model.named_parameters(), torch_fp32.named_parameters(),
                                           ref.named_parameters()):
        ok(p.grad, pt.grad, pd.grad, name)
    for (name, b), (_, bt), (_, bd) in zip(model.named_buffers(), torch_fp32.named_buffers(), ref.named_buffers()):
        if b.dtype.is_floating_point:
            ok(b, bt, bd, name)
