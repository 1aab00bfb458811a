"""One fwd+bwd of each ResNet-20 basic-block shape at B = 128 on the fp32
native path (convolutions with fused BatchNorm statistics, bn_act forward
and backward) — the launches `ncu --set full` profiles for
profiles/r2_cnn_kernels_ncu.txt (tools/ncu_cnn.sh)."""

from __future__ import annotations

import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2203_06638_b200.objectives import _Basic  # noqa: E402

CL = torch.channels_last
torch.manual_seed(0)
for cin, cout, stride, hw in ((16, 16, 1, 32), (16, 32, 2, 32), (32, 32, 1, 16), (32, 64, 2, 16), (64, 64, 1, 8)):
    blk = _Basic(cin, cout, stride).cuda().to(memory_format=CL)
    x = torch.randn(128, cin, hw, hw, device="cuda").to(memory_format=CL).requires_grad_()
    for _ in range(int(__import__("os").environ.get("LPP_ITERS", "2"))):
        y = blk(x)
        y.backward(torch.ones_like(y))
    torch.cuda.synchronize()
print("ok")
