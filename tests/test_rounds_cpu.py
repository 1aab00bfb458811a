"""The averaging-round protocol's control block is a ring (rounds.py):
far more rounds than ring cells, rounds aligned across workers, exactly the
last round unanimous, the fences of every round complete — on CPU with
host threads standing in for the Q averagers (engine.py:385-453)."""

from __future__ import annotations

import threading

from paper_2203_06638_b200.rounds import RoundControl, averager_loop


def _run_group(Q: int, slots: int, period: int):
    ctrl = RoundControl(Q)
    counters = [0] * Q
    lock = threading.Lock()
    joined = [[] for _ in range(Q)]
    final_flags = [[] for _ in range(Q)]
    fence_ok = [True] * Q
    errors = []

    def worker(q):
        try:
            # a fake updater: the slot counter advances by one per poll
            def read_counter():
                with lock:
                    if counters[q] < slots:
                        counters[q] += 1
                    return counters[q]

            def do_round(r, final, s_cur):
                fence_ok[q] &= ctrl.fence(0, r)
                fence_ok[q] &= ctrl.fence(1, r)
                joined[q].append(r)

            def on_round(r, s_cur, k_delta, unanimous):
                final_flags[q].append(unanimous)

            averager_loop(ctrl, workers=Q, read_counter=read_counter,
                          local_drained=lambda: counters[q] >= slots,
                          sync_period=lambda s: period, do_round=do_round, on_round=on_round)
        except BaseException as exc:  # pragma: no cover
            errors.append(exc)
            ctrl.abort.store(1)

    ths = [threading.Thread(target=worker, args=(q,)) for q in range(Q)]
    for t in ths:
        t.start()
    for t in ths:
        t.join(120)
    assert not errors
    return ctrl, joined, final_flags, fence_ok


def test_ring_control_runs_many_more_rounds_than_cells():
    Q = 3
    ctrl, joined, finals, fence_ok = _run_group(Q, slots=400, period=1)
    n = len(joined[0])
    assert n > 10 * RoundControl.RING
    assert all(j == list(range(1, n + 1)) for j in joined)
    assert all(f == [False] * (n - 1) + [True] for f in finals)
    assert all(fence_ok)
    # the block is fixed-size, independent of the number of rounds
    assert ctrl.buf.shape[0] == RoundControl.cells()


def test_ring_release_zeroes_the_previous_round():
    ctrl = RoundControl(2)
    for r in (1, 2):
        ctrl.vote(r, final=False)
        ctrl.vote(r, final=r == 2)
        ctrl.buf[ctrl._fence_cell(0, r)] = 2      # both workers passed fence 0
    assert ctrl.wait_votes(1) is False
    assert ctrl.wait_votes(2) is False          # one final vote of two
    # round 1's cells were released by round 2's completion
    assert ctrl.buf[ctrl._vote_cell(1)] == 0 and ctrl.buf[ctrl._fence_cell(0, 1)] == 0
    assert ctrl.buf[ctrl._vote_cell(2)] == 2
