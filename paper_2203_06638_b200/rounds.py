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
            then four arrays of RING cells, indexed by round mod RING: vote
            count, final-vote count, and the two fences (stamps published /
            quiescent; every owner's shard done)

    Rounds run in lock step (a worker votes in round r + 1 only after all Q
    votes of round r are in), so round r's cells are free again once all
    votes of round r + 1 are in: ``release(r + 1)`` zeroes them, and with
    RING >= 3 they are zero before round r + RING can use them.  Any number
    of rounds fits in a fixed-size block (no per-run round ceiling).
    """

    HEADER = 16
    STAMPS = 8
    RING = 8
    ARRAYS = 4

    def __init__(self, workers: int, max_rounds: int | None = None, buf: np.ndarray | None = None):
        self.workers = int(workers)
        # a capacity hint for per-round records only; the block is a ring
        self.max_rounds = None if max_rounds is None else int(max_rounds)
        self.ring = self.RING
        n = self.cells()
        if buf is None:
            buf = np.zeros(n, dtype=np.int64)
        if buf.dtype != np.int64 or buf.shape[0] < n:
            raise ValueError("control buffer too small")
        self.buf = buf
        self.round_calls = _Cell(buf, 0)
        self.stop = _Cell(buf, 1)
        self.abort = _Cell(buf, 2)
        self.drained = _Cell(buf, 3)

    @staticmethod
    def cells(max_rounds: int | None = None) -> int:
        return RoundControl.HEADER + RoundControl.ARRAYS * RoundControl.RING

    @staticmethod
    def nbytes(max_rounds: int | None = None) -> int:
        return 8 * RoundControl.cells()

    def publish_stamp(self, q: int, u: int) -> None:
        N.atomic_store(self.buf, self.STAMPS + q, u)

    def stamps(self) -> list[int]:
        return [N.atomic_load(self.buf, self.STAMPS + q) for q in range(self.workers)]

    def _vote_cell(self, r: int) -> int:
        return self.HEADER + r % self.RING

    def _final_cell(self, r: int) -> int:
        return self.HEADER + self.RING + r % self.RING

    def _fence_cell(self, which: int, r: int) -> int:
        return self.HEADER + (2 + which) * self.RING + r % self.RING

    def fence(self, which: int, r: int) -> bool:
        """Group-wide barrier number ``which`` (0/1) of round r; False on abort."""
        c = self._fence_cell(which, r)
        N.atomic_fetch_add(self.buf, c, 1)
        return N.atomic_wait_ge(self.buf, c, self.workers, self.buf, 2) is not None

    def vote(self, r: int, final: bool) -> None:
        if final:
            N.atomic_fetch_add(self.buf, self._final_cell(r), 1)
        N.atomic_fetch_add(self.buf, self._vote_cell(r), 1)

    def wait_votes(self, r: int) -> bool | None:
        """Block (GIL released) until all workers voted in round r.

        Returns whether the round was unanimously final; None on abort."""
        got = N.atomic_wait_ge(self.buf, self._vote_cell(r), self.workers, self.buf, 2)
        if got is None:
            return None
        unanimous = N.atomic_load(self.buf, self._final_cell(r)) == self.workers
        self.release(r)
        return unanimous

    def release(self, r: int) -> None:
        """All votes of round r are in, so nobody reads round r - 1's cells
        any more: zero them for round r - 1 + RING (idempotent)."""
        if r > 1:
            for c in (self._vote_cell(r - 1), self._final_cell(r - 1), self._fence_cell(0, r - 1),
                      self._fence_cell(1, r - 1)):
                N.atomic_store(self.buf, c, 0)


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
