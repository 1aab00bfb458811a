"""ORACLE (test infrastructure only): seeded synthetic datasets.

Restates ``make_blobs`` (/root/reference/pkg/src/asyncsgd/data.py:34-52) so
that parity inputs can be regenerated on the GPU box, where /root/reference
does not exist.  Pinned bitwise by tests/golden/data.npz.
"""

from __future__ import annotations

import numpy as np


def make_blobs(n_samples: int, n_features: int, n_classes: int, separation: float,
               noise: float, seed: int) -> tuple[np.ndarray, np.ndarray]:
    """Gaussian class blobs; labels cycle 0..k-1 (data.py:34-52)."""
    if n_samples <= 0:
        raise ValueError("need at least one sample")
    if n_classes < 2 or n_features < 1:
        raise ValueError("need >= 2 classes and >= 1 feature")
    gen = np.random.default_rng(np.random.SeedSequence([seed, n_classes, n_features]))
    centers = gen.normal(size=(n_classes, n_features))                      # data.py:48
    norms = np.maximum(np.linalg.norm(centers, axis=1, keepdims=True), 1e-12)
    centers *= separation / norms                                             # data.py:49
    y = np.arange(n_samples, dtype=np.int64) % n_classes                      # data.py:50
    X = centers[y] + noise * gen.normal(size=(n_samples, n_features))         # data.py:51
    return X, y


def cifar_blobs(n_samples: int = 2048, seed: int = 11) -> tuple[np.ndarray, np.ndarray]:
    """Config C0's CIFAR-10-shaped blobs: f=3072, k=10."""
    return make_blobs(n_samples, 3072, 10, 2.5, 0.5, seed)
