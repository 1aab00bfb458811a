"""The library's fp32 3x3 convolutions (csrc/conv_f32.cu) vs cuDNN fp32
(TF32 off) at the ResNet-20 shapes, B = 128: error against an fp64
reference for both, and time per launch (forward, dgrad, wgrad)."""

from __future__ import annotations

import sys
from pathlib import Path

import torch
import torch.nn.functional as F

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2203_06638_b200 import conv  # noqa: E402

torch.backends.cudnn.benchmark = True
torch.backends.cudnn.allow_tf32 = False
CL = torch.channels_last


def timeit(fn, n=20):
    """Device time per call: n calls captured in one CUDA graph, replayed
    (no host launch overhead in the number — these kernels are µs-scale)."""
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for _ in range(3):
            fn()
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(n):
            fn()
    g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(5):
        g.replay()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / (5 * n) * 1e3


def rel(a, ref):
    return float((a.double() - ref).abs().max() / ref.abs().max())


def main(B=128):
    g = torch.Generator(device="cuda").manual_seed(0)
    tot_n = tot_c = 0.0
    for c, hw, cnt in ((16, 32, 6), (32, 16, 5), (64, 8, 5)):
        x = torch.randn(B, c, hw, hw, device="cuda", generator=g).to(memory_format=CL)
        w = (torch.randn(c, c, 3, 3, device="cuda", generator=g) / (3 * c ** 0.5)).to(memory_format=CL)
        gy = torch.randn(B, c, hw, hw, device="cuda", generator=g).to(memory_format=CL)
        xd, wd, gyd = x.double(), w.double(), gy.double()
        y_ref = F.conv2d(xd, wd, padding=1)
        gx_ref, gw_ref, _ = torch.ops.aten.convolution_backward(gyd, xd, wd, None, (1, 1), (1, 1), (1, 1), False,
                                                                (0, 0), 1, (True, True, False))
        y_c = F.conv2d(x, w, padding=1)
        gx_c, gw_c, _ = torch.ops.aten.convolution_backward(gy, x, w, None, (1, 1), (1, 1), (1, 1), False, (0, 0),
                                                            1, (True, True, False))
        y_n = conv.conv_fwd(x, w)
        gx_n = conv.conv_fwd(gy, w, dgrad=True)
        gw_n = conv.conv_wgrad(x, gy, w)
        print(f"C={c} H=W={hw}: rel err vs fp64 — fwd cudnn {rel(y_c, y_ref):.1e} native {rel(y_n, y_ref):.1e}; "
              f"dgrad cudnn {rel(gx_c, gx_ref):.1e} native {rel(gx_n, gx_ref):.1e}; "
              f"wgrad cudnn {rel(gw_c, gw_ref):.1e} native {rel(gw_n, gw_ref):.1e}")
        flop = 2 * B * hw * hw * c * c * 9 / 1e6
        t = {
            "fwd": (timeit(lambda: F.conv2d(x, w, padding=1)), timeit(lambda: conv.conv_fwd(x, w))),
            "dgrad": (timeit(lambda: torch.ops.aten.convolution_backward(gy, x, w, None, (1, 1), (1, 1), (1, 1),
                                                                         False, (0, 0), 1, (True, False, False))),
                      timeit(lambda: conv.conv_fwd(gy, w, dgrad=True))),
            "wgrad": (timeit(lambda: torch.ops.aten.convolution_backward(gy, x, w, None, (1, 1), (1, 1), (1, 1),
                                                                         False, (0, 0), 1, (False, True, False))),
                      timeit(lambda: conv.conv_wgrad(x, gy, w))),
        }
        for k, (tc, tn) in t.items():
            print(f"   {k:5s}: cudnn {tc:7.1f} us ({flop / tc:5.1f} TF/s)  native {tn:7.1f} us "
                  f"({flop / tn:5.1f} TF/s)  x{tc / tn:.2f}")
            tot_c += cnt * tc
            tot_n += cnt * tn
    print(f"16 stride-1 3x3 convs per minibatch (fwd+dgrad+wgrad): cudnn {tot_c:.0f} us, native {tot_n:.0f} us")
    for ci, co, hw in ((16, 32, 32), (32, 64, 16)):
        x = torch.randn(B, ci, hw, hw, device="cuda", generator=g).to(memory_format=CL)
        w = torch.randn(co, ci, 1, 1, device="cuda", generator=g).to(memory_format=CL)
        gy = torch.randn(B, co, hw // 2, hw // 2, device="cuda", generator=g).to(memory_format=CL)
        cells = conv.arrival_cells("cuda")
        cb = torch.ops.aten.convolution_backward
        t = {"fwd": (timeit(lambda: F.conv2d(x, w, stride=2)), timeit(lambda: conv.conv1x1s2(x, w, 0))),
             "dgrad": (timeit(lambda: cb(gy, x, w, None, (2, 2), (0, 0), (1, 1), False, (0, 0), 1, (True, False, False))),
                       timeit(lambda: conv.conv1x1s2(gy, w, 1))),
             "wgrad": (timeit(lambda: cb(gy, x, w, None, (2, 2), (0, 0), (1, 1), False, (0, 0), 1, (False, True, False))),
                       timeit(lambda: conv.conv1x1s2(x, w, 2, gy, cells)))}
        print(f"1x1 stride 2 {ci}->{co} at {hw}x{hw}: " + "; ".join(
            f"{k} cudnn {tc:.1f} us native {tn:.1f} us" for k, (tc, tn) in t.items()))
        w3 = torch.randn(co, ci, 3, 3, device="cuda", generator=g).to(memory_format=CL)
        t = {"fwd": (timeit(lambda: F.conv2d(x, w3, stride=2, padding=1)), timeit(lambda: conv.conv3x3s2(x, w3, 0))),
             "dgrad": (timeit(lambda: cb(gy, x, w3, None, (2, 2), (1, 1), (1, 1), False, (0, 0), 1, (True, False, False))),
                       timeit(lambda: conv.conv3x3s2(gy, w3, 1))),
             "wgrad": (timeit(lambda: cb(gy, x, w3, None, (2, 2), (1, 1), (1, 1), False, (0, 0), 1, (False, True, False))),
                       timeit(lambda: conv.conv3x3s2(x, w3, 2, gy, cells)))}
        print(f"3x3 stride 2 {ci}->{co} at {hw}x{hw}: " + "; ".join(
            f"{k} cudnn {tc:.1f} us native {tn:.1f} us" for k, (tc, tn) in t.items()))


if __name__ == "__main__":
    main()
