"""ORACLE (test infrastructure only): the small CNN of BASELINE config 0 in
fp64 on the CPU.

The reference has no CNN; its engine takes any ``Objective``
(objectives.py:33-63), and config 0 plugs a small CNN into it.  This module
is that objective restated independently of the product: the network is
written with ``torch.nn.functional`` in float64 over the reference flat
layout ``[conv1.w (O,I,kh,kw), conv1.b, conv2.w, conv2.b, fc.w (out,in),
fc.b]``, and ``grad_block`` is the gradient of the mean batch loss sliced
to the block (objectives.py:286-308 semantics; autograd restricted to the
block's tensors).  Pinned by a finite-difference check
(tests/test_oracle_golden.py, the reference's test_objectives.py:56-73
criterion) and by tests/golden/serialized_cnn_lpp.npz /
engine_cnn_q1u1.npz (the reference's own engine and schedule primitives
driving this objective).
"""

from __future__ import annotations

import numpy as np
import torch
import torch.nn as nn
import torch.nn.functional as F

SHAPES = ((16, 3, 3, 3), (16,), (32, 16, 3, 3), (32,), (10, 512), (10,))
LAYER_COUNTS = tuple(int(np.prod(s)) for s in SHAPES)


def make_images(n: int, seed: int, n_classes: int = 10, pattern_scale: float = 0.0):
    """Synthetic CIFAR-shaped data: labels, then N(0,1) images, one torch CPU
    generator seeded ``seed`` (the product's host-data generator); with
    ``pattern_scale`` > 0 every image also gets its class's fixed random
    pattern (a second generator seeded ``seed + 7919``) times the scale —
    make_blobs (data.py:34-52) in image space, a learnable task."""
    g = torch.Generator().manual_seed(seed)
    labels = torch.randint(0, n_classes, (n,), generator=g)
    images = torch.randn(n, 3, 32, 32, generator=g)
    if pattern_scale:
        pg = torch.Generator().manual_seed(seed + 7919)
        images += (torch.randn(n_classes, 3, 32, 32, generator=pg) * pattern_scale)[labels]
    return images.double().numpy(), labels.numpy()


class SmallCnnOracle:
    def __init__(self, features, labels):
        self.features = torch.as_tensor(np.asarray(features, dtype=np.float64))
        self.labels = torch.as_tensor(np.asarray(labels), dtype=torch.long)
        self.n_samples = int(self.features.shape[0])
        self.layer_param_counts = LAYER_COUNTS
        self.edges = tuple(int(v) for v in np.concatenate([[0], np.cumsum(LAYER_COUNTS)]))
        self.dim = self.edges[-1]

    def init_params(self, seed: int) -> np.ndarray:
        """torch's default Conv2d/Linear init under ``manual_seed(seed)``, in
        construction order (conv1, conv2, fc)."""
        torch.manual_seed(seed)
        mods = [nn.Conv2d(3, 16, 3, stride=2, padding=1), nn.Conv2d(16, 32, 3, stride=2, padding=1),
                nn.Linear(512, 10)]
        return torch.cat([p.detach().reshape(-1) for m in mods for p in m.parameters()]).double().numpy()

    def _params(self, x):
        xt = torch.as_tensor(np.asarray(x, dtype=np.float64))
        return [xt[self.edges[i]:self.edges[i + 1]].view(SHAPES[i]).clone() for i in range(6)]

    def _loss(self, ps, batch):
        xb = self.features[torch.as_tensor(np.asarray(batch), dtype=torch.long)]
        yb = self.labels[torch.as_tensor(np.asarray(batch), dtype=torch.long)]
        h = torch.tanh(F.conv2d(xb, ps[0], ps[1], stride=2, padding=1))
        h = torch.tanh(F.conv2d(h, ps[2], ps[3], stride=2, padding=1))
        logits = F.linear(F.avg_pool2d(h, 2).flatten(1), ps[4], ps[5])
        return F.cross_entropy(logits, yb)

    def loss(self, x, batch) -> float:
        with torch.no_grad():
            return float(self._loss(self._params(x), batch))

    def grad_block(self, x, lo, hi, batch) -> np.ndarray:
        first = self.edges.index(lo)
        last = self.edges.index(hi) - 1
        ps = self._params(x)
        leaves = ps[first:last + 1]
        for p in leaves:
            p.requires_grad_(True)
        grads = torch.autograd.grad(self._loss(ps, batch), leaves)
        return torch.cat([g.reshape(-1) for g in grads]).numpy()
