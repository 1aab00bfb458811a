"""ORACLE (test infrastructure only): NDJSON event log reader and the
deterministic round replay.

Restates ``load_event_log`` (/root/reference/pkg/src/asyncsgd/instrumentation.py:424-463)
and ``replay_rounds`` (instrumentation.py:166-219): write stamps order each
worker's model writes, averaging stamps cut that order into rounds; every
worker's view starts at the previous round mean and applies its logged
block updates (``view[lo:lo+len] -= lr * grad``) in write-stamp order, and
the next mean is the fixed-order average of the final views.  A GPU run
written with ``paper_2203_06638_b200.eventlog.save_event_log`` replays
here against its own measured round means.  Pinned on a log written by the
reference itself (tests/golden/eventlog_ref.ndjson.gz).
"""

from __future__ import annotations

import bisect
import gzip
import json
from dataclasses import dataclass
from pathlib import Path

import numpy as np


@dataclass
class Update:
    worker: int
    rank: int
    s: int
    u: int
    k_claim: int
    block_id: int
    lr: float
    clean: object
    tags: object
    grad: object
    snapshot: object


@dataclass
class Stamp:
    worker: int
    round: int
    u: int
    s_cur: int
    k_delta: int
    snapshot: object
    mean: object


def load_event_log(path) -> tuple[list[Update], list[Stamp]]:
    path = Path(path)
    opener = gzip.open if path.suffix == ".gz" else open
    ups, sts = [], []

    def arr(v, dt=np.float64):
        return None if v is None else np.asarray(v, dtype=dt)

    with opener(path, "rt") as fh:
        for line in fh:
            o = json.loads(line)
            if o["kind"] == "update":
                ups.append(Update(o["worker"], o["rank"], o["s"], o["u"], o["k_claim"], o["block_id"],
                                  o["lr"], o["clean"], arr(o["tags"], np.int64), arr(o["grad"]),
                                  arr(o["snapshot"])))
            else:
                sts.append(Stamp(o["worker"], o["round"], o["u"], o["s_cur"], o["k_delta"],
                                 arr(o["snapshot"]), arr(o["mean"])))
    return ups, sts


def replay_rounds(updates, stamps, x0: np.ndarray, boundaries) -> dict:
    """Round means (index 0 = x0), per-update view distances and clean flags."""
    by_w: dict[int, list] = {}
    for st in stamps:
        by_w.setdefault(st.worker, []).append(st)
    for v in by_w.values():
        v.sort(key=lambda st: st.u)
    recs: dict[int, list] = {}
    for r in updates:
        recs.setdefault(r.worker, []).append(r)
    for v in recs.values():
        v.sort(key=lambda r: r.u)
    counts = {q: len(v) for q, v in by_w.items()}
    if len(set(counts.values())) > 1:
        raise ValueError(f"unaligned round counts {counts}")
    rounds = next(iter(counts.values()), 0)
    workers = sorted(by_w)
    grouped = {}
    for q in workers:
        orders = [st.u for st in by_w[q]]
        per = [[] for _ in range(rounds + 1)]
        for r in recs.get(q, []):
            per[bisect.bisect_left(orders, r.u)].append(r)
        if per[rounds]:
            raise ValueError("updates recorded after the final round")
        grouped[q] = per
    dim = x0.shape[0]
    means = [np.asarray(x0, dtype=np.float64).copy()]
    dists = []
    for j in range(rounds):
        finals = np.empty((len(workers), dim))
        for qi, q in enumerate(workers):
            view = means[-1].copy()
            start = by_w[q][j - 1].u if j > 0 else 0
            for r in grouped[q][j]:
                gap = view - r.snapshot
                clean = None if r.tags is None else bool((r.tags >= start).all())
                dists.append((r.u, float(np.sqrt(gap @ gap)), clean))
                lo = 0 if r.block_id == 0 else boundaries[r.block_id - 1]
                view[lo:lo + len(r.grad)] -= r.lr * r.grad
            finals[qi] = view
        means.append(np.mean(finals, axis=0))
    dists.sort(key=lambda d: d[0])
    return {"round_means": means, "distances": np.array([d[1] for d in dists]),
            "clean": np.array([d[2] for d in dists], dtype=object),
            "k_bar": max((st.k_delta for st in stamps), default=0)}
