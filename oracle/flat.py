"""ORACLE (test infrastructure only): the reference's desk-scale objectives.

Restates ``QuadraticObjective`` (objectives.py:111-145: gradient = x minus
the batch's mean target, sliced) and ``LogisticObjective``
(objectives.py:152-193: margin = s * (f @ x), gradient = f^T (-s / (1 +
exp(margin))) / n, sliced).  Pinned by tests/golden/serialized_quad8_lpp.npz
and serialized_logreg8_lap.npz (serialized runs built from the reference).
"""

from __future__ import annotations

import numpy as np


class QuadOracle:
    def __init__(self, targets):
        self.targets = np.asarray(targets, dtype=np.float64)
        self.n_samples, self.dim = self.targets.shape

    def init_params(self, seed):
        return np.zeros(self.dim)

    def grad_block(self, x, lo, hi, batch):
        return (x - self.targets[batch].mean(axis=0))[lo:hi]


class LogisticOracle:
    def __init__(self, features, labels01):
        self.features = np.asarray(features, dtype=np.float64)
        self.signs = np.where(np.asarray(labels01) == 1, 1.0, -1.0)
        self.n_samples, self.dim = self.features.shape

    def init_params(self, seed):
        return np.zeros(self.dim)

    def grad_block(self, x, lo, hi, batch):
        f = self.features[batch]
        s = self.signs[batch]
        w = -s / (1.0 + np.exp(s * (f @ x)))
        return (f.T @ w / len(batch))[lo:hi]


def make_linear_targets(n_samples, dim, spread, noise, seed):
    """data.py:55-66."""
    gen = np.random.default_rng(np.random.SeedSequence([seed, dim]))
    center = spread * gen.normal(size=dim)
    return center + noise * gen.normal(size=(n_samples, dim))
