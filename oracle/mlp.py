"""ORACLE (test infrastructure only): the reference MLP objective, in numpy.

Restates ``MlpObjective`` (/root/reference/pkg/src/asyncsgd/objectives.py:200-319):
fully connected net, tanh hidden layers, softmax cross-entropy head, flat
layout ``[W1, b1, W2, b2, ...]`` with ``W_l`` of shape (in, out) and
``z = a @ W + b`` (objectives.py:203-205, 242-250, 264-274).  The truncated
backward of ``grad_block`` walks from the output down to the block's
input-most layer only (objectives.py:286-308).

``dtype`` selects fp64 (the reference) or fp32 (used to measure the
fp32-vs-fp64 gap that sets the parity tolerance).  Pinned against the
reference by tests/golden/mlp.npz.
"""

from __future__ import annotations

import numpy as np


class MlpOracle:
    def __init__(self, features: np.ndarray, labels: np.ndarray, hidden: tuple[int, ...],
                 n_classes: int, dtype=np.float64):
        self.dtype = np.dtype(dtype)
        self.features = np.asarray(features, dtype=self.dtype)
        self.labels = np.asarray(labels, dtype=np.int64)
        self.n_samples = self.features.shape[0]
        self.widths = (self.features.shape[1], *hidden, n_classes)
        self.n_layers = len(self.widths) - 1
        self.layer_param_counts = tuple(
            self.widths[l] * self.widths[l + 1] + self.widths[l + 1] for l in range(self.n_layers)
        )
        self.dim = int(sum(self.layer_param_counts))
        self.edges = tuple(int(v) for v in np.concatenate([[0], np.cumsum(self.layer_param_counts)]))
        self.onehot = np.eye(n_classes, dtype=self.dtype)[self.labels]

    # objectives.py:235-240 — per-layer normal(scale=1/sqrt(fan_in)) weights, zero biases
    def init_params(self, seed: int) -> np.ndarray:
        gen = np.random.default_rng(np.random.SeedSequence([seed, self.dim]))
        x = np.zeros(self.dim)
        for l, (w, _b) in enumerate(self.views(x)):
            w[:] = gen.normal(scale=1.0 / np.sqrt(self.widths[l]), size=w.shape)
        return x.astype(self.dtype, copy=False)

    def views(self, x: np.ndarray):
        out = []
        for l in range(self.n_layers):
            lo, hi = self.edges[l], self.edges[l + 1]
            a, b = self.widths[l], self.widths[l + 1]
            out.append((x[lo : lo + a * b].reshape(a, b), x[lo + a * b : hi]))
        return out

    def first_layer_of(self, start: int, stop: int) -> int:
        if start == 0 and stop == self.dim:
            return 0
        if start not in self.edges or stop not in self.edges:
            raise ValueError(f"block ({start}, {stop}) does not align to layer boundaries")
        return self.edges.index(start)

    def forward(self, x: np.ndarray, batch: np.ndarray):
        acts = [self.features[batch]]
        z = None
        layers = self.views(x)
        for l, (w, b) in enumerate(layers):
            z = acts[-1] @ w + b
            if l < self.n_layers - 1:
                acts.append(np.tanh(z))
        shifted = z - z.max(axis=1, keepdims=True)
        logp = shifted - np.log(np.exp(shifted).sum(axis=1, keepdims=True))
        return acts, logp

    def loss(self, x: np.ndarray, batch: np.ndarray) -> float:
        _, logp = self.forward(x, batch)
        return -float(logp[np.arange(len(batch)), self.labels[batch]].mean())

    def grad_block(self, x: np.ndarray, start: int, stop: int, batch: np.ndarray) -> np.ndarray:
        """Gradient restricted to [start, stop) via the truncated backward."""
        first = self.first_layer_of(start, stop)
        acts, logp = self.forward(x, batch)
        layers = self.views(x)
        n = len(batch)
        g = np.zeros(self.dim, dtype=self.dtype)
        gl = self.views(g)
        delta = (np.exp(logp) - self.onehot[batch]) / n
        for l in range(self.n_layers - 1, first - 1, -1):
            w, _ = layers[l]
            gw, gb = gl[l]
            gw[:] = acts[l].T @ delta
            gb[:] = delta.sum(axis=0)
            delta = delta @ w.T
            if l - 1 >= first:
                delta = delta * (1.0 - acts[l] * acts[l])
        return g[start:stop]

    def backward_cost(self, start: int, stop: int) -> int:
        first = self.first_layer_of(start, stop)
        return sum(2 * self.widths[l] * self.widths[l + 1] for l in range(first, self.n_layers))
