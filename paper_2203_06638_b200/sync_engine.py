"""Synchronous baselines B1 / B2 (engine.py:544-629): MB-SGD and PL-SGD with
one CUDA-graph step per worker; the collective is NCCL all-reduce (AVG) in a
one-process-per-GPU group and a fixed-order K4 mean in one process."""

from __future__ import annotations

import time

import numpy as np
import torch

from . import _native as N
from .arena import Arena, enable_peer_access
from .partition import Block
from .records import RunConfig
from .schedules import lr_at, sync_every
from .step import StepProgram


# ---------------------------------------------------------------------------
# synchronous baselines (B1 MB-SGD, B2 PL-SGD) — engine.py:544-629


class _SyncEngine:
    """MB-SGD / PL-SGD with one CUDA-graph step per worker; the collective
    is NCCL all-reduce in a multi-process group and a fixed-order K4 mean in
    one process."""

    def __init__(self, cfg: RunConfig, group=None, host_batches: bool = False):
        self.cfg = cfg
        obj = cfg.objective
        self.dim = obj.dim
        self.group = group
        self.host_batches = host_batches
        self.x0_host = np.asarray(obj.init_params(cfg.seed), dtype=np.float64)
        x0 = torch.from_numpy(self.x0_host.astype(np.float32))
        devs = cfg.devices or (torch.cuda.current_device(),)
        self.local = [group.rank] if group is not None else list(range(cfg.workers))
        self.dev_of = {q: (torch.cuda.current_device() if group is not None else devs[q % len(devs)])
                       for q in self.local}
        self.x = {q: Arena(self.dim, self.dev_of[q]) for q in self.local}
        self.g = {q: Arena(self.dim, self.dev_of[q]) for q in self.local}
        self.m = {q: Arena(self.dim, self.dev_of[q]) for q in self.local} if cfg.momentum else {}
        self.gmean = {q: torch.zeros(self.dim + 4, device=f"cuda:{self.dev_of[q]}") for q in self.local}
        self.stream = {}
        self.prog = {}
        full = {0: Block(0, self.dim)}
        for q in self.local:
            self.x[q].tensor.copy_(x0)
            with torch.cuda.device(self.dev_of[q]):
                self.stream[q] = torch.cuda.Stream()
                self.prog[q] = StepProgram(obj, torch.device("cuda", self.dev_of[q]), self.x[q].tensor,
                                           self.g[q].tensor, full, cfg.batch_size, self.stream[q],
                                           input_mode="batch" if host_batches else
                                           ("random" if cfg.sampling == "device" else "index"),
                                           use_graphs=cfg.use_graphs, seed=cfg.seed + q)
        if group is None and len(set(self.dev_of.values())) > 1:
            for a in self.local:
                for b in self.local:
                    if self.dev_of[a] != self.dev_of[b]:
                        enable_peer_access(self.dev_of[a], self.dev_of[b])
        # pinned staging ring for the host-drawn indices: slot k % depth is
        # rewritten only after the copy that last read it has completed
        self.depth = 4
        self.idx_pinned = torch.zeros((self.depth, cfg.workers, cfg.batch_size), dtype=torch.long,
                                      pin_memory=True)
        self.slot_events = [[None] * self.depth for _ in range(cfg.workers)]
        self.k = 0
        torch.cuda.synchronize()

    def _grads(self, shards: np.ndarray | None):
        cfg = self.cfg
        slot = self.k % self.depth
        self.k += 1
        for q in self.local:
            st = self.stream[q]
            with torch.cuda.stream(st):
                ev = self.slot_events[q][slot]
                if ev is not None:
                    ev.synchronize()
                if shards is not None:
                    idx = shards[q * cfg.batch_size:(q + 1) * cfg.batch_size]
                    if self.host_batches:
                        t = torch.from_numpy(idx)
                        self.prog[q].xb.copy_(cfg.objective.features.index_select(0, t).pin_memory(),
                                              non_blocking=True)
                        self.prog[q].yb.copy_(cfg.objective.labels.index_select(0, t), non_blocking=True)
                    else:
                        self.idx_pinned[slot, q].copy_(torch.from_numpy(idx))
                        self.prog[q].idx.copy_(self.idx_pinned[slot, q], non_blocking=True)
                self.prog[q].run(0)
                ev = torch.cuda.Event()
                ev.record(st)
                self.slot_events[q][slot] = ev

    def _apply(self, q, grad_ptr, lr):
        cfg = self.cfg
        N.apply_sgd(self.x[q].ptr, grad_ptr, self.m[q].ptr if cfg.momentum else None, self.dim,
                    float(lr), None, cfg.momentum, cfg.weight_decay, N.MODES[cfg.apply_mode],
                    self.stream[q].cuda_stream)

    def _mean_grads(self):
        """mean_q g_q (engine.py:568) into gmean (fixed order in one process)."""
        if self.group is not None:
            q = self.group.rank
            with torch.cuda.stream(self.stream[q]):
                t = self.g[q].tensor
                self.group.allreduce_mean(t)
            return {q: self.g[q].ptr}
        for q in self.local:
            self.stream[q].synchronize()
        q0 = self.local[0]
        s0 = self.stream[q0]
        with torch.cuda.device(self.dev_of[q0]), torch.cuda.stream(s0):
            N.average_shard([self.g[q].ptr for q in range(self.cfg.workers)], 0, self.dim,
                            self.gmean[q0].data_ptr(), N.MODE_PLAIN, s0.cuda_stream)
            ptrs = {}
            for q in self.local:
                if self.dev_of[q] == self.dev_of[q0]:
                    ptrs[q] = self.gmean[q0].data_ptr()
                else:
                    # cross-device copy ordered after the mean on s0
                    self.gmean[q][: self.dim].copy_(self.gmean[q0][: self.dim])
                    ptrs[q] = self.gmean[q].data_ptr()
        # every worker's apply (on its own stream) after the mean and the copies
        s0.synchronize()
        return ptrs

    def _mean_params(self):
        if self.group is not None:
            q = self.group.rank
            with torch.cuda.stream(self.stream[q]):
                self.group.allreduce_mean(self.x[q].tensor)
            return
        for q in self.local:
            self.stream[q].synchronize()
        q0 = self.local[0]
        s0 = self.stream[q0]
        with torch.cuda.device(self.dev_of[q0]), torch.cuda.stream(s0):
            # x_q = mean exactly (xs[:] = mean, engine.py:612): write the mean,
            # then copy it into every arena, all on s0 (ordered after the mean)
            N.average_shard([self.x[q].ptr for q in range(self.cfg.workers)], 0, self.dim,
                            self.gmean[q0].data_ptr(), N.MODE_PLAIN, s0.cuda_stream)
            for q in self.local:
                self.x[q].tensor.copy_(self.gmean[q0][: self.dim])
        # the next _grads on every stream[q] reads x[q]: finish the copies first
        s0.synchronize()

    def run(self, steps: int | None = None) -> float:
        cfg = self.cfg
        steps = cfg.budget if steps is None else steps
        gen = np.random.default_rng(np.random.SeedSequence([cfg.seed, 0, 1]))
        n = cfg.objective.n_samples
        since = 0
        self.rounds = 0
        starts = {}
        for q in self.local:
            torch.cuda.synchronize(self.dev_of[q])
            e = torch.cuda.Event(enable_timing=True)
            e.record(self.stream[q])
            starts[q] = e
        self.t0 = time.perf_counter()
        self.evals = []
        last_eval = 0
        for k in range(1, steps + 1):
            lr = lr_at(cfg.lr, k - 1)
            shards = gen.integers(0, n, cfg.workers * cfg.batch_size) if cfg.sampling == "host" else None
            self._grads(shards)
            if cfg.algo == "mb_sgd":
                if cfg.workers == 1 and self.group is None:
                    self._apply(0, self.g[0].ptr, lr)
                else:
                    ptrs = self._mean_grads()
                    for q in self.local:
                        self._apply(q, ptrs[q], lr)
                if cfg.eval_interval and k % cfg.eval_interval == 0:     # engine.py:569-570
                    self.evals.append((k, k, (time.perf_counter() - self.t0) * 1e3, 0,
                                       self.x[self.local[0]].tensor.clone()))
            else:
                for q in self.local:
                    self._apply(q, self.g[q].ptr, lr)
                since += 1
                if since >= sync_every(cfg.sync, k) or k == steps:
                    if cfg.workers > 1:
                        self._mean_params()
                    self.rounds += 1
                    since = 0
                    if cfg.eval_interval and k >= last_eval + cfg.eval_interval:  # engine.py:615-616
                        last_eval = k
                        self.evals.append((k, self.rounds, (time.perf_counter() - self.t0) * 1e3, 0,
                                           self.x[self.local[0]].tensor.clone()))
        ms = 0.0
        for q in self.local:
            e = torch.cuda.Event(enable_timing=True)
            e.record(self.stream[q])
            e.synchronize()
            ms = max(ms, starts[q].elapsed_time(e))
        self.wall_ms = (time.perf_counter() - self.t0) * 1e3
        return ms

    def final_values(self) -> np.ndarray:
        return self.x[self.local[0]].tensor.cpu().numpy()

    def close(self) -> None:
        """Free graphs and arenas now (see ``_Worker.close``)."""
        torch.cuda.synchronize()
        for p in self.prog.values():
            p.close()
        self.prog = {}
        for a in [*self.x.values(), *self.g.values(), *self.m.values()]:
            a.close()
