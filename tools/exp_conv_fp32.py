"""cuDNN fp32 (TF32 off) convolution time per ResNet-20 shape, standalone,
channels-last, B = 128: forward, dgrad, wgrad, and the FFMA throughput each
reaches (2 * MACs / time).  Decides whether hand-written fp32 convolutions
could move the fp32 headline."""

from __future__ import annotations

import torch
import torch.nn.functional as F

torch.backends.cudnn.benchmark = True
torch.backends.cudnn.allow_tf32 = False
torch.backends.cuda.matmul.allow_tf32 = False

B = 128
# (cin, cout, hw_in, stride, k, count in ResNet-20)
SHAPES = [(3, 16, 32, 1, 3, 1), (16, 16, 32, 1, 3, 6), (16, 32, 32, 2, 3, 1), (16, 32, 32, 2, 1, 1),
          (32, 32, 16, 1, 3, 5), (32, 64, 16, 2, 3, 1), (32, 64, 16, 2, 1, 1), (64, 64, 8, 1, 3, 5)]


def timeit(fn, n=50):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n * 1e3


def main():
    dev = torch.device("cuda")
    tot = {"fwd": 0.0, "dgrad": 0.0, "wgrad": 0.0}
    macs_tot = 0
    print(f"{'cin':>4}{'cout':>5}{'hw':>4}{'s':>2}{'k':>2}{'n':>3} | {'fwd us':>8}{'TF/s':>6} | {'dgrad':>8}{'TF/s':>6} | {'wgrad':>8}{'TF/s':>6}")
    for cin, cout, hw, s, k, cnt in SHAPES:
        x = torch.randn(B, cin, hw, hw, device=dev).to(memory_format=torch.channels_last)
        w = torch.randn(cout, cin, k, k, device=dev).to(memory_format=torch.channels_last)
        pad = k // 2
        y = F.conv2d(x, w, stride=s, padding=pad)
        gy = torch.randn_like(y)
        ho = y.shape[2]
        macs = B * ho * ho * cout * cin * k * k
        t_f = timeit(lambda: F.conv2d(x, w, stride=s, padding=pad))
        t_d = timeit(lambda: torch.ops.aten.convolution_backward(gy, x, w, None, (s, s), (pad, pad), (1, 1),
                                                                  False, (0, 0), 1, (True, False, False)))
        t_w = timeit(lambda: torch.ops.aten.convolution_backward(gy, x, w, None, (s, s), (pad, pad), (1, 1),
                                                                  False, (0, 0), 1, (False, True, False)))
        f = 2 * macs / 1e6
        print(f"{cin:>4}{cout:>5}{hw:>4}{s:>2}{k:>2}{cnt:>3} | {t_f:8.1f}{f / t_f:6.1f} | {t_d:8.1f}{f / t_d:6.1f} | "
              f"{t_w:8.1f}{f / t_w:6.1f}")
        tot["fwd"] += cnt * t_f
        tot["dgrad"] += cnt * t_d if cin != 3 else 0.0
        tot["wgrad"] += cnt * t_w
        macs_tot += cnt * macs
    s = sum(tot.values())
    print(f"ResNet-20 convs per minibatch of {B}: fwd {tot['fwd']:.0f} us, dgrad {tot['dgrad']:.0f} us, "
          f"wgrad {tot['wgrad']:.0f} us, total {s:.0f} us; {3 * 2 * macs_tot / s / 1e6:.1f} TFLOP/s; "
          f"conv-only ceiling {B / s * 1e6:,.0f} images/s")


if __name__ == "__main__":
    main()
