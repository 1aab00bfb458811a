"""ORACLE (test infrastructure / CPU baseline only): threaded CPU port of the
reference engine's asynchronous path, for the bench's ``cpu_baseline`` leg
and ``bench.py --impl reference``.

It follows ``_run_async`` (/root/reference/pkg/src/asyncsgd/engine.py:466-523)
thread for thread over an fp64 numpy store whose element ops are the
REFERENCE's own compiled ``_atomics`` (oracle/_ref, built by oracle/Makefile
from /root/reference/pkg/src/asyncsgd/_atomics.c) when present:

* updaters (engine.py:315-383): cooperative pacing while a round is due,
  claim slot (``fetch_add_i64``), lr (schedules.py:56-68), PASSM+ block
  (partition.py:132-145), 16 sampled write tags drawn first then gathered
  (``gather_i64``), per-element snapshot (``snapshot_f64``), block gradient,
  tagged CAS apply (``accum_cas_tagged_f64``), clean classification;
* averagers (engine.py:385-453): poll, open/join rounds, snapshot, slot-
  deposit mean all-reduce through a ``threading.Barrier`` (engine.py:199-229),
  tagged ``add_assign(mean - snapshot)``, unanimous-final exit.

The reference has no CNN objective, so the block gradient of the bench's
ResNet-20 workload is computed with torch on the CPU (autograd restricted
to the block's leaf tensors), one model replica per updater,
with momentum 0.9 / weight decay 5e-4 applied per updater before the CAS
apply like the GPU arm.
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


def _select(s: int, t_st: int, rank: int) -> int:
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


class _Ops:
    """The reference's compiled _atomics, or numpy stand-ins."""

    def __init__(self):
        self.mod = native.reference_atomics()
        self.kind = "reference" if self.mod is not None else "port"
        self._lock = threading.Lock()

    def fetch_add(self, cell: np.ndarray, delta: int = 1) -> int:
        if self.mod is not None:
            return int(self.mod.fetch_add_i64(cell, 0, delta))
        with self._lock:
            v = int(cell[0])
            cell[0] = v + delta
            return v

    def load(self, cell: np.ndarray) -> int:
        return int(self.mod.load_i64(cell, 0)) if self.mod is not None else int(cell[0])

    def store(self, cell: np.ndarray, v: int) -> None:
        if self.mod is not None:
            self.mod.store_i64(cell, 0, v)
        else:
            cell[0] = v

    def snapshot(self, src, out):
        if self.mod is not None:
            self.mod.snapshot_f64(src, out)
        else:
            out[:] = src

    def gather(self, tags, idx, out):
        if self.mod is not None:
            self.mod.gather_i64(tags, idx, out)
        else:
            out[:] = tags[idx]

    def accum_tagged(self, dst, tags, start, delta, scale, stamp):
        if self.mod is not None:
            self.mod.accum_cas_tagged_f64(dst, tags, start, delta, scale, stamp)
        else:
            dst[start:start + len(delta)] += scale * delta
            tags[start:start + len(delta)] = stamp


def _balanced(sizes: list[int], k: int) -> list[int]:
    """balanced_boundaries with non-negative costs (partition.py:86-129)."""
    edges = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)

    def count(start, cap):
        c, acc = 0, None
        for s in sizes[start:]:
            if s > cap:
                return 1 << 60
            if acc is None or acc + s > cap:
                c, acc = c + 1, s
            else:
                acc += s
        return c

    lo, hi = max(sizes), int(edges[-1])
    while lo < hi:
        mid = (lo + hi) // 2
        lo, hi = (lo, mid) if count(0, mid) <= k else (mid + 1, hi)
    cuts, start = [0], 0
    for rem in range(k, 1, -1):
        for c in range(start + 1, len(sizes) - rem + 2):
            if edges[c] - edges[start] > lo:
                break
            if count(c, lo) <= rem - 1:
                cuts.append(c)
                start = c
                break
    cuts.append(len(sizes))
    return [int(edges[c]) for c in cuts]


def run_lpp_cpu(slots: int, updaters: int = 4, batch_size: int = 128, n_samples: int = 4096,
                threads: int | None = None, seed: int = 0, momentum: float = 0.9,
                weight_decay: float = 5e-4, workers: int = 1, period: int = 16,
                tag_sample: int = 16) -> dict:
    """LPP-SGD on ResNet-20 / CIFAR-10-shaped synthetic data, CPU only.

    ``slots`` is the per-worker budget (claim-then-process: ``slots +
    updaters`` minibatches per worker).  Returns images, seconds, cores, the
    atomics kind, rounds and p_hat.
    """
    import torch

    cores = threads or len(os.sched_getaffinity(0))
    torch.set_num_threads(cores)
    ops = _Ops()
    Net = _resnet20(torch)
    torch.manual_seed(seed)
    template = Net()
    sizes = [p.numel() for p in template.parameters()]
    edges = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    dim = int(edges[-1])
    bounds = _balanced(sizes, updaters)
    x0 = torch.cat([p.detach().reshape(-1) for p in template.parameters()]).double().numpy()
    gen = torch.Generator().manual_seed(seed)
    X = torch.randn(n_samples, 3, 32, 32, generator=gen)
    Y = torch.randint(0, 10, (n_samples,), generator=gen)
    t_st = max(1, slots // 10)
    total = slots + updaters
    switch = total // 2

    class Worker:
        def __init__(self):
            self.values = x0.copy()
            self.tags = np.zeros(dim, dtype=np.int64)
            self.counter = np.zeros(1, dtype=np.int64)
            self.order = np.zeros(1, dtype=np.int64)
            self.last_avg = np.zeros(1, dtype=np.int64)
            self.synced_at = np.zeros(1, dtype=np.int64)
            self.exited = np.zeros(1, dtype=np.int64)

    ws = [Worker() for _ in range(workers)]
    stop = np.zeros(1, dtype=np.int64)
    round_gate = np.zeros(1, dtype=np.int64)
    round_calls = np.zeros(1, dtype=np.int64)
    stats = {"done": 0, "clean": 0, "classified": 0, "rounds": 0}
    lock = threading.Lock()
    errors: list = []
    slots_mat = np.zeros((workers, dim))
    flags = np.zeros(workers, dtype=bool)
    mean_buf = np.zeros(dim)
    unanimous_box = [False]
    barrier = threading.Barrier(workers)

    def sync_every(s):
        return 1 if s < switch else period

    # every updater's model is built before the clock starts; each updater
    # thread runs its intra-op work on its share of the cores (OpenMP's
    # thread count is per calling thread: without this, U threads x all cores)
    models = {(q, r): Net() for q in range(workers) for r in range(1, updaters + 1)}
    per_thread = max(1, cores // (updaters * workers))

    def updater(q: int, rank: int):
        w = ws[q]
        try:
            torch.set_num_threads(per_thread)
            model = models[(q, rank)]
            params = list(model.parameters())
            snap = np.empty(dim)
            mom = np.zeros(dim) if momentum else None
            rng = np.random.default_rng(np.random.SeedSequence([seed, q, rank]))
            tag_out = np.empty(tag_sample, dtype=np.int64)
            s = 0
            while s < slots and not ops.load(stop):
                # cooperative pacing (engine.py:325-335)
                while not ops.load(stop):
                    if ops.load(round_gate) == 0:
                        s_now = ops.load(w.counter)
                        if s_now - ops.load(w.synced_at) < sync_every(s_now):
                            break
                    time.sleep(5e-5)
                s = ops.fetch_add(w.counter)
                lr = _lr(0.1, 0.25, t_st, total, s)
                b = _select(s, t_st, rank)
                blo, bhi = (0, dim) if b == 0 else (bounds[b - 1], bounds[b])
                idx = np.sort(rng.choice(dim, size=tag_sample, replace=False))
                ops.gather(w.tags, idx, tag_out)
                ops.snapshot(w.values, snap)
                flat = torch.from_numpy(snap).float()
                with torch.no_grad():
                    for i, p in enumerate(params):
                        p.copy_(flat[edges[i]:edges[i + 1]].view_as(p))
                first = int(np.searchsorted(edges, blo, side="right") - 1)
                last = int(np.searchsorted(edges, bhi, side="left") - 1)
                bidx = torch.from_numpy(rng.integers(0, n_samples, batch_size))
                loss = torch.nn.functional.cross_entropy(model(X[bidx]), Y[bidx])
                grads = torch.autograd.grad(loss, params[first:last + 1])
                g = torch.cat([t.reshape(-1) for t in grads]).double().numpy()
                if weight_decay:
                    g = g + weight_decay * snap[blo:bhi]
                if mom is not None:
                    mom[blo:bhi] = momentum * mom[blo:bhi] + g
                    g = mom[blo:bhi]
                k_claim = ops.load(w.last_avg)
                u = ops.fetch_add(w.order) + 1
                ops.accum_tagged(w.values, w.tags, blo, lr * g, -1.0, u)
                clean = bool((tag_out >= k_claim).all())
                with lock:
                    stats["done"] += 1
                    stats["classified"] += 1
                    stats["clean"] += int(clean)
        except BaseException as exc:  # pragma: no cover - surfaced below
            errors.append(exc)
            ops.store(stop, 1)
            barrier.abort()
        finally:
            ops.fetch_add(w.exited)

    def averager(q: int):
        w = ws[q]
        s_pre, round_no, backoff = 0, 0, 0.0
        snap = np.empty(dim)
        try:
            while True:
                s_cur = ops.load(w.counter)
                drain = ops.load(w.exited) == updaters
                pending = ops.load(round_calls) > round_no
                fresh = s_cur - s_pre >= sync_every(s_cur)
                if not (drain or fresh) and not pending:
                    time.sleep(backoff)
                    backoff = min(2e-4, backoff * 2 + 1e-5)
                    continue
                if drain and not fresh and not pending:
                    time.sleep(2e-3)
                    pending = ops.load(round_calls) > round_no
                if not pending:
                    ops.fetch_add(round_calls)
                backoff = 0.0
                ops.fetch_add(round_gate)
                try:
                    ops.snapshot(w.values, snap)
                    # _MeanAllReduce.reduce (engine.py:216-226)
                    slots_mat[q] = snap
                    flags[q] = drain
                    if barrier.wait() == 0:
                        np.mean(slots_mat, axis=0, out=mean_buf)
                        unanimous_box[0] = bool(flags.all())
                    barrier.wait()
                    mean = mean_buf.copy()
                    unanimous = unanimous_box[0]
                    barrier.wait()
                    u_avg = ops.fetch_add(w.order) + 1
                    ops.accum_tagged(w.values, w.tags, 0, mean - snap, 1.0, u_avg)
                    ops.store(w.last_avg, u_avg)
                    ops.store(w.synced_at, s_cur)
                finally:
                    ops.fetch_add(round_gate, -1)
                round_no += 1
                s_pre = s_cur
                if unanimous:
                    with lock:
                        stats["rounds"] = max(stats["rounds"], round_no)
                    return
        except threading.BrokenBarrierError:
            return
        except BaseException as exc:  # pragma: no cover
            errors.append(exc)
            ops.store(stop, 1)
            barrier.abort()

    ths = [threading.Thread(target=averager, args=(q,)) for q in range(workers)]
    ths += [threading.Thread(target=updater, args=(q, r)) for q in range(workers)
            for r in range(1, updaters + 1)]
    t0 = time.perf_counter()
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    sec = time.perf_counter() - t0
    if errors:
        raise errors[0]
    return {"images": stats["done"] * batch_size, "seconds": sec, "cores": cores,
            "atomics": ops.kind, "minibatches": stats["done"], "dim": dim,
            "rounds": stats["rounds"],
            "p_hat": stats["clean"] / stats["classified"] if stats["classified"] else 1.0,
            "finite": bool(np.all(np.isfinite(ws[0].values)))}
