"""Averaging-round protocol of a worker group (host side of K4).

Restates the reference's averager control flow (``_averager_body``,
/root/reference/pkg/src/asyncsgd/engine.py:385-453) for a group whose
workers are CUDA devices (or processes) instead of threads:

* a round is due for worker q when ``s_cur - s_pre >= sync_every(s_cur)``
  (engine.py:395-401); any worker's trigger opens the round for all
  (``round_calls``, engine.py:399-412) — opening is a CAS so exactly one
  opener wins per round;
* each worker joins every opened round, runs its share of the data plane
  (the owner-computes K4 launch over its shard) and votes whether it is
  drained (all its updaters exited);
* averagers — never updaters — wait for all Q votes of the round; the group
  stops after the first round in which every vote is final (the unanimous
  drain round of engine.py:452-453).  A drained worker with nothing new does
  not open rounds on its own until every worker is drained (the reference
  sleeps 2 ms for the same purpose, engine.py:406-410).

The control block is an int64 array: a numpy buffer for in-process groups
or a POSIX shared-memory segment for one-process-per-GPU groups; all cells
are accessed with the C ABI's host atomics (K6).  Pure host code: it is
exercised on CPU by the multi-process gloo tests.
"""

from __future__ import annotations

import time

import numpy as np

from . import _native as N


class _Cell:
    """One int64 cell of the control block (address resolved once)."""

    __slots__ = ("_b", "_a")

    def __init__(self, buf, i):
        self._b = buf                      # keeps the buffer alive
        self._a = N.cell_address(buf, i)

    def read(self) -> int:
        return N.lib.lpp_atomic_load_i64(self._a)

    def add(self, d: int) -> int:
        return N.lib.lpp_atomic_fetch_add_i64(self._a, d)

    def store(self, v: int) -> None:
        N.lib.lpp_atomic_store_i64(self._a, v)

    def cas(self, expected: int, desired: int) -> bool:
        return bool(N.lib.lpp_atomic_cas_i64(self._a, expected, desired))


class RoundControl:
    """Cells shared by a group's averagers.

    layout: [0] round_calls  [1] stop  [2] abort  [3] drained workers
            [8 : 16]  each worker's update-order stamp for the current round
                      (the owners write it into every arena's tags, K5)
            then four per-round arrays of R+2 cells: vote count, final-vote
            count, and the two fences (all published/paused; all shards done)
    """

    HEADER = 16
    STAMPS = 8

    def __init__(self, workers: int, max_rounds: int, buf: np.ndarray | None = None):
        self.workers = int(workers)
        self.max_rounds = int(max_rounds)
        n = self.cells(max_rounds)
        if buf is None:
            buf = np.zeros(n, dtype=np.int64)
        if buf.dtype != np.int64 or buf.shape[0] < n:
            raise ValueError("control buffer too small")
        self.buf = buf
        self.round_calls = _Cell(buf, 0)
        self.stop = _Cell(buf, 1)
        self.abort = _Cell(buf, 2)
        self.drained = _Cell(buf, 3)

    ARRAYS = 4

    @staticmethod
    def cells(max_rounds: int) -> int:
        return RoundControl.HEADER + RoundControl.ARRAYS * (int(max_rounds) + 2)

    @staticmethod
    def nbytes(max_rounds: int) -> int:
        return 8 * RoundControl.cells(max_rounds)

    def publish_stamp(self, q: int, u: int) -> None:
        N.atomic_store(self.buf, self.STAMPS + q, u)

    def stamps(self) -> list[int]:
        return [N.atomic_load(self.buf, self.STAMPS + q) for q in range(self.workers)]

    def _final_cell(self, r: int) -> int:
        return self.HEADER + self.max_rounds + 2 + r

    def _fence_cell(self, which: int, r: int) -> int:
        return self.HEADER + (2 + which) * (self.max_rounds + 2) + r

    def fence(self, which: int, r: int) -> bool:
        """Group-wide barrier number ``which`` (0/1) of round r; False on abort."""
        c = self._fence_cell(which, r)
        N.atomic_fetch_add(self.buf, c, 1)
        return N.atomic_wait_ge(self.buf, c, self.workers, self.buf, 2) is not None

    def vote(self, r: int, final: bool) -> None:
        if r > self.max_rounds:
            self.abort.store(1)
            raise RuntimeError("averaging round budget of the control block exceeded")
        if final:
            N.atomic_fetch_add(self.buf, self._final_cell(r), 1)
        N.atomic_fetch_add(self.buf, self.HEADER + r, 1)

    def wait_votes(self, r: int) -> bool | None:
        """Block (GIL released) until all workers voted in round r.

        Returns whether the round was unanimously final; None on abort."""
        got = N.atomic_wait_ge(self.buf, self.HEADER + r, self.workers, self.buf, 2)
        if got is None:
            return None
        return N.atomic_load(self.buf, self._final_cell(r)) == self.workers


def averager_loop(ctrl: RoundControl, *, workers: int, read_counter, local_drained, sync_period,
                  do_round, on_round, stop_after: int | None = None,
                  max_backoff: float = 2e-4) -> int:
    """Run one worker's averager until the group's unanimous final round.

    read_counter()            -> this worker's slot counter C^q
    local_drained()           -> all of this worker's updaters have exited
    sync_period(s)            -> sync_every(scheme, s)
    do_round(r, final, s_cur) -> run this worker's share of round r (blocking)
    on_round(r, s_cur, k_delta, unanimous) -> bookkeeping after the vote
    Returns the number of rounds joined.
    """
    s_pre, round_no, backoff = 0, 0, 0.0
    while True:
        if ctrl.abort.read():
            return round_no
        s_cur = read_counter()
        drain = bool(local_drained())
        pending = ctrl.round_calls.read() > round_no
        fresh = s_cur - s_pre >= sync_period(s_cur)
        if not pending:
            if fresh or (drain and ctrl.drained.read() == workers):
                ctrl.round_calls.cas(round_no, round_no + 1)
            else:
                time.sleep(backoff)
                backoff = min(max_backoff, backoff * 2 + 1e-5)
                continue
        backoff = 0.0
        r = round_no + 1
        ctrl.vote(r, drain)
        do_round(r, drain, s_cur)
        unanimous = ctrl.wait_votes(r)
        if unanimous is None:
            return round_no
        round_no = r
        if stop_after is not None and round_no >= stop_after:
            ctrl.stop.store(1)
        on_round(r, s_cur, s_cur - s_pre, unanimous)
        s_pre = s_cur
        if unanimous:
            return round_no
