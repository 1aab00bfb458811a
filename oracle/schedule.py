"""ORACLE (test infrastructure only): canonical serialized LPP/LAP-SGD schedule.

The reference's live async runs are not deterministic (round
counts and slot->rank pairings vary run to run), so parity is defined on a
*canonical serialized schedule* that both this oracle and the CUDA engine's
``schedule="serialized"`` mode follow exactly.  It is the reference's
Algorithm-1 engine (engine.py:315-383 updater step, :385-453 averager round)
with the thread interleaving fixed:

    x_q = init(seed); C_q = 0; s_pre_q = 0
    rng[q][r] = default_rng(SeedSequence([seed, q, r]))        engine.py:293
    repeat sweeps:
      for q in 0..Q-1, for r in 1..U (if still active):
        s = C_q; C_q += 1                                       engine.py:336
        lr = lr_at(sched, s)                                    engine.py:337
        b  = select_block(s, T_st, nblocks, r) if lpp else 0    engine.py:338-342
        batch = rng[q][r].integers(0, n, B)                     engine.py:351 (record "full": no tag draw)
        x_q[b] -= lr * grad_block(x_q, b, batch)                engine.py:352-355
        if s >= budget: deactivate (q, r)                       claim-then-process, engine.py:321
      if any_q C_q - s_pre_q >= sync_every(C_q) or all inactive:  engine.py:395-401
        m = mean_q x_q (fixed q order); x_q += m - x_q          engine.py:418-421, 219-220
        s_pre_q = C_q; round += 1
        stop after the round in which every updater is inactive   engine.py:452-453
    final_values = m of the last round                          engine.py:507

Extensions for the configuration bench.py times (B200 side):
``mu``/``wd`` give every updater its own momentum buffer m[q][r] over the
whole arena and apply, per element of the block, in the kernels' operation
order (oracle/apply_ref.c ``sgd_delta``; the momentum / weight-decay
extension point SPEC.md:382,385):  g' = g + wd*x;  m = mu*m + g';
x += -(lr*m).  ``tag_draw=k`` reproduces record modes other than "full":
the updater's rng first draws ``rng.choice(d, k, replace=False)`` tag
indices, then the batch (engine.py:343-351).  ``batch_fn(q, r, t)`` replaces
the numpy batch stream with another index stream (e.g. the device sampler
restated in oracle/devsample.py), t = the updater's local step count.

The scalar schedule helpers are restated here (not imported from the
product package) so the checker is independent of the checked code:
select_block (partition.py:132-145), lr_at (schedules.py:56-68),
sync_every (schedules.py:93-95).  Pinned bitwise against reference
primitives by tests/golden/serialized_*.npz.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np


# --- scalar schedule restatements -------------------------------------------


def select_block(s: int, t_st: int, num_blocks: int, rank: int) -> int:
    if not 1 <= rank <= num_blocks:
        raise ValueError(f"rank {rank} outside [1, {num_blocks}]")
    if s <= t_st or (s - t_st) % 2 == 1:
        return 0
    return rank


@dataclass(frozen=True)
class Lr:
    kind: str
    alpha0: float
    total: int
    warmup: int = 0
    peak: float = 0.0
    milestones: tuple = ()
    gamma: float = 0.1

    def at(self, s: int) -> float:
        if s < self.warmup:
            return self.alpha0 + (self.peak - self.alpha0) * s / self.warmup
        if self.kind == "cosine":
            if s >= self.total:
                return 0.0
            span = self.total - self.warmup
            return self.peak * 0.5 * (1.0 + math.cos(math.pi * (s - self.warmup) / span))
        return self.peak * self.gamma ** sum(1 for m in self.milestones if s >= m)


def sync_every(s_cur: int, switch_point: int, period: int) -> int:
    return 1 if s_cur < switch_point else period


# --- the serialized run -------------------------------------------------------


@dataclass
class SerializedTrace:
    final_values: np.ndarray
    xs: list                       # per-worker arenas at the end
    block_ids: list = field(default_factory=list)   # (q, rank, s, block_id)
    lrs: list = field(default_factory=list)         # (q, rank, s, lr)
    rounds: list = field(default_factory=list)      # (round, sweep, (C_q...))
    counter_finals: list = field(default_factory=list)
    losses: list = field(default_factory=list)      # (q, rank, s, loss at the step's snapshot)


class EpochSampler:
    """objectives.py:77-104: per-epoch reshuffled walk over an index shard."""

    def __init__(self, indices, seed):
        self.ix, self.seed, self.epoch, self.pos = np.asarray(indices), seed, -1, 0
        self.perm = self.ix[:0]

    def next_batch(self, b):
        out = np.empty(b, dtype=np.int64)
        f = 0
        while f < b:
            if self.pos >= len(self.perm):
                self.epoch += 1
                g = np.random.default_rng(np.random.SeedSequence([self.seed, self.epoch]))
                self.perm = self.ix[g.permutation(len(self.ix))]
                self.pos = 0
            k = min(b - f, len(self.perm) - self.pos)
            out[f:f + k] = self.perm[self.pos:self.pos + k]
            self.pos += k
            f += k
        return out


def run_serialized(obj, *, algo: str, workers: int, updaters: int, boundaries: tuple,
                   lr: Lr, switch_point: int, period: int, budget: int, warm_start: int,
                   batch_size: int, seed: int, dtype=np.float64,
                   epoch_partition: bool = False, mu: float = 0.0, wd: float = 0.0,
                   tag_draw: int = 0, batch_fn=None, record_loss: bool = False) -> SerializedTrace:
    """Run the canonical schedule; ``obj`` has init_params/grad_block(x, lo, hi, batch)."""
    if algo not in ("lap_sgd", "lpp_sgd"):
        raise ValueError("serialized schedule covers the asynchronous algorithms")
    dim = obj.dim
    nblocks = len(boundaries) - 1
    x0 = np.asarray(obj.init_params(seed), dtype=dtype)
    xs = [x0.copy() for _ in range(workers)]
    counters = [0] * workers
    s_pre = [0] * workers
    gens = [[np.random.default_rng(np.random.SeedSequence([seed, q, r]))
             for r in range(1, updaters + 1)] for q in range(workers)]
    active = [[True] * updaters for _ in range(workers)]
    # engine.py:294-296: shard arange(n)[q::Q], seed seed*1000 + q*10 + rank
    samplers = [[EpochSampler(np.arange(obj.n_samples)[q::workers], seed * 1000 + q * 10 + r)
                 for r in range(1, updaters + 1)] for q in range(workers)] if epoch_partition else None
    moms = [[np.zeros(dim, dtype=dtype) for _ in range(updaters)] for _ in range(workers)] if mu else None
    local_t = [[0] * updaters for _ in range(workers)]
    trace = SerializedTrace(final_values=x0.copy(), xs=xs)
    sweep = 0
    mean = x0.copy()
    while True:
        for q in range(workers):
            for ri in range(updaters):
                if not active[q][ri]:
                    continue
                rank = ri + 1
                s = counters[q]
                counters[q] += 1
                step_lr = lr.at(s)
                b = select_block(s, warm_start, nblocks, rank) if algo == "lpp_sgd" else 0
                lo, hi = (0, dim) if b == 0 else (boundaries[b - 1], boundaries[b])
                if tag_draw:
                    gens[q][ri].choice(dim, size=min(tag_draw, dim), replace=False)
                if batch_fn is not None:
                    batch = batch_fn(q, ri, local_t[q][ri])
                elif samplers is not None:
                    batch = samplers[q][ri].next_batch(batch_size)
                else:
                    batch = gens[q][ri].integers(0, obj.n_samples, batch_size)
                local_t[q][ri] += 1
                if record_loss:
                    trace.losses.append((q, rank, s, obj.loss(xs[q], batch)))
                g = obj.grad_block(xs[q], lo, hi, batch)
                if mu or wd:
                    g = np.asarray(g, dtype=dtype)
                    if wd:
                        g = g + dtype(wd) * xs[q][lo:hi]
                    if mu:
                        m = moms[q][ri]
                        m[lo:hi] = dtype(mu) * m[lo:hi] + g
                        g = m[lo:hi]
                if dtype == np.float32:
                    delta = np.float32(step_lr) * g.astype(np.float32)
                else:
                    delta = step_lr * g
                xs[q][lo:hi] += -delta          # ParamStore.sub_assign: dst += -1 * delta
                trace.block_ids.append((q, rank, s, b))
                trace.lrs.append((q, rank, s, step_lr))
                if s >= budget:
                    active[q][ri] = False
        sweep += 1
        drained = not any(a for row in active for a in row)
        fresh = any(counters[q] - s_pre[q] >= sync_every(counters[q], switch_point, period)
                    for q in range(workers))
        if fresh or drained:
            stacked = np.stack(xs)
            mean = np.mean(stacked, axis=0)
            for q in range(workers):
                xs[q] += mean - xs[q]
                s_pre[q] = counters[q]
            trace.rounds.append((len(trace.rounds) + 1, sweep, tuple(counters)))
        if drained:
            break
    trace.final_values = mean.copy()
    trace.counter_finals = list(counters)
    return trace
