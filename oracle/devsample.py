"""ORACLE (test infrastructure only): restatement of the B200 device batch
samplers, so that runs drawing their minibatches on the GPU
(``RunConfig.sampling="device"``, the configuration bench.py times) can be
replayed by the serialized oracle (oracle/schedule.py ``batch_fn``).

The device sampler is the build's own i.i.d. stream (the reference draws
``rng.integers(0, n, B)`` on the host, engine.py:351); it is specified in
paper_2203_06638_b200/csrc/updater.cu (``sample_one``): for updater key k
and local step t, element i of the batch is

    base = splitmix64(k ^ splitmix64(t))
    r    = splitmix64(base + i * 0xD1B54A32D192ED03)      (mod 2^64)
    idx  = (r * n) >> 64                                  (128-bit product)

This file restates that formula independently in Python integers (no
product code is imported); tests/test_bench_config_gpu.py checks the GPU
engine against the oracle driven by it.
"""

from __future__ import annotations

import numpy as np

M64 = (1 << 64) - 1


def splitmix64(z: int) -> int:
    z = (z + 0x9E3779B97F4A7C15) & M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return z ^ (z >> 31)


def iid_batch(key: int, step: int, batch: int, n: int) -> np.ndarray:
    key &= M64
    base = splitmix64(key ^ splitmix64(step & M64))
    out = np.empty(batch, dtype=np.int64)
    for i in range(batch):
        r = splitmix64((base + i * 0xD1B54A32D192ED03) & M64)
        out[i] = (r * n) >> 64
    return out


def engine_key(seed: int, q: int, r: int) -> int:
    """The key the engine gives updater r (0-based) of worker q
    (paper_2203_06638_b200/async_engine.py, ``StepProgram(seed=...)``)."""
    return seed * 7919 + q * 101 + r + 1
