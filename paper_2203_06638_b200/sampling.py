"""Minibatch index sampling (a9), host side.

Same streams as the reference (``/root/reference/pkg/src/asyncsgd/objectives.py:70-104``):

* ``sample_batch(rng, n, B)`` — uniform i.i.d. with replacement,
  ``rng.integers(0, n, B)`` (objectives.py:70-74);
* ``EpochSampler(indices, seed)`` — walks a per-epoch reshuffled permutation
  of a worker's index shard, epoch e permuted by
  ``default_rng(SeedSequence([seed, e]))`` (objectives.py:77-104); the engine
  gives updater ``rank`` of worker q the shard ``arange(n)[q::Q]`` and seed
  ``seed*1000 + q*10 + rank`` (engine.py:294-296), the paper's reshuffled
  partition sampling.

Indices are drawn on the host and copied to the device with the step
(pinned ring), so the device sees exactly the reference's batches.
"""

from __future__ import annotations

import numpy as np


def sample_batch(rng: np.random.Generator, n_samples: int, batch_size: int) -> np.ndarray:
    if n_samples <= 0 or batch_size <= 0:
        raise ValueError("need positive sample count and batch size")
    return rng.integers(0, n_samples, size=batch_size)


class EpochSampler:
    def __init__(self, indices, seed: int):
        idx = np.asarray(indices)
        if idx.size == 0:
            raise ValueError("empty shard")
        self._indices = idx
        self._seed = seed
        self._epoch = -1
        self._order = idx[:0]
        self._pos = 0

    def _next_epoch(self) -> None:
        self._epoch += 1
        gen = np.random.default_rng(np.random.SeedSequence([self._seed, self._epoch]))
        self._order = self._indices[gen.permutation(len(self._indices))]
        self._pos = 0

    def next_batch(self, batch_size: int) -> np.ndarray:
        out = np.empty(batch_size, dtype=np.int64)
        got = 0
        while got < batch_size:
            if self._pos >= len(self._order):
                self._next_epoch()
            take = min(batch_size - got, len(self._order) - self._pos)
            out[got:got + take] = self._order[self._pos:self._pos + take]
            self._pos += take
            got += take
        return out


def worker_sampler(n_samples: int, workers: int, q: int, rank: int, seed: int) -> EpochSampler:
    """The epoch-partition sampler of updater ``rank`` of worker ``q`` (engine.py:294-296)."""
    return EpochSampler(np.arange(n_samples)[q::workers], seed=seed * 1000 + q * 10 + rank)
