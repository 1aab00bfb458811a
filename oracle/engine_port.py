"""ORACLE (test infrastructure / CPU baseline only): threaded CPU port of the
reference engine's asynchronous path, for the bench's ``cpu_baseline`` leg
and ``bench.py --impl reference``.

It follows ``_updater_loop`` (/root/reference/pkg/src/asyncsgd/engine.py:315-383)
step for step — claim slot (``fetch_add_i64``), lr (schedules.py:56-68),
PASSM+ block (partition.py:132-145), per-element snapshot (``snapshot_f64``),
block gradient, CAS apply (``accum_cas_f64``) — over an fp64 numpy store,
using the REFERENCE's own compiled ``_atomics`` (oracle/_ref, built from
/root/reference/pkg/src/asyncsgd/_atomics.c by oracle/Makefile) when it is
present, else numpy stand-ins.  The reference has no CNN objective, so the
block gradient of the bench's ResNet-20 workload is computed with torch on
the CPU (autograd restricted to the block's leaf tensors, as PAPER.md:190),
one model replica per updater thread.

Workers: Q = 1 here (the CPU figure is a single-host baseline); averaging
at Q = 1 is an exact no-op (test_engine.py:169-182), so it is skipped.
"""

from __future__ import annotations

import math
import os
import threading
import time

import numpy as np

from . import native


def _lr(alpha0: float, peak: float, warmup: int, total: int, s: int) -> float:
    if s < warmup:
        return alpha0 + (peak - alpha0) * s / warmup
    if s >= total:
        return 0.0
    return peak * 0.5 * (1.0 + math.cos(math.pi * (s - warmup) / (total - warmup)))


def _select(s: int, t_st: int, nblocks: int, rank: int) -> int:
    if s <= t_st or (s - t_st) % 2 == 1:
        return 0
    return rank


def _resnet20(torch):
    nn, F = torch.nn, torch.nn.functional

    class Basic(nn.Module):
        def __init__(self, cin, cout, stride):
            super().__init__()
            self.c1 = nn.Conv2d(cin, cout, 3, stride, 1, bias=False)
            self.b1 = nn.BatchNorm2d(cout)
            self.c2 = nn.Conv2d(cout, cout, 3, 1, 1, bias=False)
            self.b2 = nn.BatchNorm2d(cout)
            self.sc = None
            if stride != 1 or cin != cout:
                self.sc = nn.Sequential(nn.Conv2d(cin, cout, 1, stride, bias=False), nn.BatchNorm2d(cout))

        def forward(self, x):
            o = F.relu(self.b1(self.c1(x)))
            o = self.b2(self.c2(o))
            return F.relu(o + (x if self.sc is None else self.sc(x)))

    class Net(nn.Module):
        def __init__(self):
            super().__init__()
            self.c = nn.Conv2d(3, 16, 3, 1, 1, bias=False)
            self.b = nn.BatchNorm2d(16)
            blocks, cin = [], 16
            for cout, st in ((16, 1), (32, 2), (64, 2)):
                for i in range(3):
                    blocks.append(Basic(cin, cout, st if i == 0 else 1))
                    cin = cout
            self.blocks = nn.Sequential(*blocks)
            self.fc = nn.Linear(64, 10)

        def forward(self, x):
            o = F.relu(self.b(self.c(x)))
            o = self.blocks(o)
            return self.fc(F.adaptive_avg_pool2d(o, 1).flatten(1))

    return Net


class _Atomics:
    """The reference's compiled _atomics, or numpy stand-ins."""

    def __init__(self):
        self.mod = native.reference_atomics()
        self.kind = "reference" if self.mod is not None else "port"
        self._lock = threading.Lock()

    def fetch_add(self, cell: np.ndarray) -> int:
        if self.mod is not None:
            return int(self.mod.fetch_add_i64(cell, 0, 1))
        with self._lock:
            v = int(cell[0])
            cell[0] = v + 1
            return v

    def snapshot(self, src: np.ndarray, out: np.ndarray) -> None:
        if self.mod is not None:
            self.mod.snapshot_f64(src, out)
        else:
            out[:] = src

    def sub(self, dst: np.ndarray, start: int, delta: np.ndarray) -> None:
        if self.mod is not None:
            self.mod.accum_cas_f64(dst, start, delta, -1.0)
        else:
            dst[start:start + len(delta)] -= delta


def run_lpp_cpu(slots: int, updaters: int = 4, batch_size: int = 128, n_samples: int = 4096,
                threads: int | None = None, seed: int = 0, momentum: float = 0.9,
                weight_decay: float = 5e-4) -> dict:
    """LPP-SGD on ResNet-20 / CIFAR-10-shaped synthetic data, CPU only.

    Returns images, seconds, cores and the atomics kind.  ``slots`` is the
    per-worker budget (claim-then-process: ``slots + updaters`` minibatches).
    Momentum / weight decay are applied per updater before the CAS apply,
    matching the GPU arm's per-stream momentum semantics.
    """
    import torch

    cores = threads or len(os.sched_getaffinity(0))
    torch.set_num_threads(cores)
    at = _Atomics()
    Net = _resnet20(torch)
    torch.manual_seed(seed)
    template = Net()
    sizes = [p.numel() for p in template.parameters()]
    edges = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    dim = int(edges[-1])
    # layer-aligned U-block split minimising the worst block size (the
    # reference balanced_boundaries with non-negative costs)
    k = updaters
    lo, hi = max(sizes), dim
    def nblocks(cap):
        c, acc = 0, None
        for s in sizes:
            if acc is None or acc + s > cap:
                c, acc = c + 1, s
            else:
                acc += s
        return c
    while lo < hi:
        mid = (lo + hi) // 2
        lo, hi = (lo, mid) if nblocks(mid) <= k else (mid + 1, hi)
    cap, cuts, start = lo, [0], 0
    for rem in range(k, 1, -1):
        for c in range(start + 1, len(sizes) - rem + 2):
            if edges[c] - edges[start] > cap:
                break
            tail = sizes[c:]
            cnt, acc = 0, None
            for s in tail:
                if acc is None or acc + s > cap:
                    cnt, acc = cnt + 1, s
                else:
                    acc += s
            if cnt <= rem - 1:
                cuts.append(c)
                start = c
                break
    cuts.append(len(sizes))
    bounds = [int(edges[c]) for c in cuts]

    values = torch.cat([p.detach().reshape(-1) for p in template.parameters()]).double().numpy().copy()
    counter = np.zeros(1, dtype=np.int64)
    gen = torch.Generator().manual_seed(seed)
    X = torch.randn(n_samples, 3, 32, 32, generator=gen)
    Y = torch.randint(0, 10, (n_samples,), generator=gen)
    t_st = max(1, slots // 10)
    total = slots + updaters
    done = [0]
    lock = threading.Lock()
    errors: list = []

    def updater(rank: int):
        try:
            model = Net()
            params = list(model.parameters())
            snap = np.empty(dim)
            mom = np.zeros(dim) if momentum else None
            rng = np.random.default_rng(np.random.SeedSequence([seed, 0, rank]))
            s = 0
            while s < slots:
                s = at.fetch_add(counter)
                lr = _lr(0.1, 0.25, t_st, total, s)
                b = _select(s, t_st, k, rank)
                blo, bhi = (0, dim) if b == 0 else (bounds[b - 1], bounds[b])
                at.snapshot(values, snap)
                flat = torch.from_numpy(snap).float()
                with torch.no_grad():
                    for i, p in enumerate(params):
                        p.copy_(flat[edges[i]:edges[i + 1]].view_as(p))
                first = int(np.searchsorted(edges, blo, side="right") - 1)
                last = int(np.searchsorted(edges, bhi, side="left") - 1)
                leaves = params[first:last + 1]
                idx = torch.from_numpy(rng.integers(0, n_samples, batch_size))
                loss = torch.nn.functional.cross_entropy(model(X[idx]), Y[idx])
                grads = torch.autograd.grad(loss, leaves)
                g = torch.cat([t.reshape(-1) for t in grads]).double().numpy()
                if weight_decay:
                    g = g + weight_decay * snap[blo:bhi]
                if mom is not None:
                    mom[blo:bhi] = momentum * mom[blo:bhi] + g
                    g = mom[blo:bhi]
                at.sub(values, blo, lr * g)
                with lock:
                    done[0] += 1
        except BaseException as exc:  # pragma: no cover - surfaced below
            errors.append(exc)

    ths = [threading.Thread(target=updater, args=(r,)) for r in range(1, updaters + 1)]
    t0 = time.perf_counter()
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    sec = time.perf_counter() - t0
    if errors:
        raise errors[0]
    return {"images": done[0] * batch_size, "seconds": sec, "cores": cores,
            "atomics": at.kind, "minibatches": done[0], "dim": dim,
            "finite": bool(np.all(np.isfinite(values)))}
