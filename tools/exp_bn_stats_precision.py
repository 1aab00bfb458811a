"""Precision of the fused BatchNorm statistics (sum, sum of squares in
fp32 partials) against fp64 statistics of the same fp32 conv output, on
post-ReLU inputs (positive channel means)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2203_06638_b200 import conv  # noqa: E402

CL = torch.channels_last
torch.manual_seed(0)
for c, hw in ((16, 32), (32, 16), (64, 8)):
    x = torch.relu(torch.randn(128, c, hw, hw, device="cuda")).to(memory_format=CL)
    w = (torch.randn(c, c, 3, 3, device="cuda") / (3 * c ** 0.5)).to(memory_format=CL)
    y, sums = conv.conv_fwd(x, w, stats=conv.arrival_cells("cuda", 2)[8:])
    yd = y.double()
    n = y.numel() / c
    mean_ref = yd.mean((0, 2, 3))
    var_ref = yd.var((0, 2, 3), unbiased=False)
    s = sums.double().view(c, 2)
    mean = s[:, 0] / n
    var = s[:, 1] / n - mean * mean
    print(f"C={c}: |mean|/std {float((mean_ref.abs() / var_ref.sqrt()).mean()):.2f}; rel err mean "
          f"{float(((mean - mean_ref).abs() / var_ref.sqrt()).max()):.1e} (of std), var "
          f"{float(((var - var_ref).abs() / var_ref).max()):.1e}")
