"""ORACLE (test infrastructure only): CIFAR ResNet-20 in fp64 on the CPU.

BASELINE config 1's network as an ``Objective`` (objectives.py:33-63) for
the serialized oracle (oracle/schedule.py), written here with
``torch.nn.functional`` only — no product module is imported.  Layout of
the flat vector (the product arena's, 65 tensors, d20 = 272,474):

    conv1.w, bn1.(w, b),
    9 basic blocks [conv1.w, bn1.(w,b), conv2.w, bn2.(w,b),
                    + (shortcut 1x1 conv.w, bn.(w,b)) where stride 2 / widening],
    fc.w (10, 64), fc.b

3x3/1x1 conv weights are stored (O, kh, kw, I) when ``channels_last``
(the product's channels-last arena layout) and (O, I, kh, kw) otherwise.
BatchNorm runs in training mode (batch statistics, eps 1e-5): the loss of a
step depends only on the parameters and the batch, as in the product's
captured step.  ``grad_block`` is the gradient of the mean cross-entropy
restricted to the block's tensors (objectives.py:286-308).
The initial vector is an input (``x0``): the oracle checks the training
trajectory from a given start.
"""

from __future__ import annotations

import numpy as np
import torch
import torch.nn.functional as F


def _layout(num_classes: int = 10):
    shapes, convs = [], []

    def conv(o, i, k):
        convs.append(len(shapes))
        shapes.append((o, i, k, k))

    def bn(c):
        shapes.extend([(c,), (c,)])

    blocks = []
    conv(16, 3, 3)
    bn(16)
    cin = 16
    for cout, stride in ((16, 1), (32, 2), (64, 2)):
        for j in range(3):
            s = stride if j == 0 else 1
            first = len(shapes)
            conv(cout, cin, 3)
            bn(cout)
            conv(cout, cout, 3)
            bn(cout)
            sc = s != 1 or cin != cout
            if sc:
                conv(cout, cin, 1)
                bn(cout)
            blocks.append((first, s, sc))
            cin = cout
    shapes.extend([(num_classes, 64), (num_classes,)])
    return shapes, set(convs), blocks


class ResNet20Oracle:
    def __init__(self, features, labels, x0, channels_last: bool = True, num_classes: int = 10):
        self.features = torch.as_tensor(np.asarray(features, dtype=np.float64))
        self.labels = torch.as_tensor(np.asarray(labels), dtype=torch.long)
        self.n_samples = int(self.features.shape[0])
        self.shapes, self.convs, self.blocks = _layout(num_classes)
        counts = [int(np.prod(s)) for s in self.shapes]
        self.layer_param_counts = tuple(counts)
        self.edges = tuple(int(v) for v in np.concatenate([[0], np.cumsum(counts)]))
        self.dim = self.edges[-1]
        self.channels_last = channels_last
        self.x0 = np.asarray(x0, dtype=np.float64)
        if self.x0.shape != (self.dim,):
            raise ValueError(f"x0 must have {self.dim} entries")

    def init_params(self, seed: int) -> np.ndarray:
        return self.x0.copy()

    def _params(self, x):
        xt = torch.as_tensor(np.asarray(x, dtype=np.float64))
        ps = []
        for i, shp in enumerate(self.shapes):
            flat = xt[self.edges[i]:self.edges[i + 1]].clone()
            ps.append(flat)
        return ps

    def _shaped(self, ps, i):
        shp = self.shapes[i]
        if i in self.convs and self.channels_last:
            o, c, kh, kw = shp
            return ps[i].view(o, kh, kw, c).permute(0, 3, 1, 2)
        return ps[i].view(shp)

    def _loss(self, ps, batch):
        idx = torch.as_tensor(np.asarray(batch), dtype=torch.long)
        h = self.features[idx]
        yb = self.labels[idx]
        W = lambda i: self._shaped(ps, i)  # noqa: E731

        def bnorm(t, i):
            return F.batch_norm(t, None, None, W(i), W(i + 1), training=True, eps=1e-5)

        h = F.relu(bnorm(F.conv2d(h, W(0), padding=1), 1))
        for first, s, sc in self.blocks:
            out = F.relu(bnorm(F.conv2d(h, W(first), stride=s, padding=1), first + 1))
            out = bnorm(F.conv2d(out, W(first + 3), padding=1), first + 4)
            short = bnorm(F.conv2d(h, W(first + 6), stride=s), first + 7) if sc else h
            h = F.relu(out + short)
        h = F.adaptive_avg_pool2d(h, 1).flatten(1)
        n = len(self.shapes)
        logits = F.linear(h, W(n - 2), W(n - 1))
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
