"""The multi-GPU group's host side on CPU: world_size-2 ``gloo`` processes
share the POSIX-shared-memory round-control block and run the averager
protocol (paper_2203_06638_b200.rounds, the restatement of
engine.py:385-453) with real updater threads bumping the slot counters.

Checked (the reference's engine invariants, test_engine.py:152-235,264-278):
every round is joined by every worker; the group stops on exactly one
unanimous final round; every rank counts the same rounds; round_budget
stops the updaters; the final-mean gather reassembles the owner shards.
"""

from __future__ import annotations

import os
import socket
import threading
import time

import torch.multiprocessing as mp


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, mode, out_q):
    import sys
    from pathlib import Path

    sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2203_06638_b200.engine import shard_bounds
    from paper_2203_06638_b200.group import ProcessGroup
    from paper_2203_06638_b200.paramstore import AtomicCounter
    from paper_2203_06638_b200.rounds import averager_loop

    budget, U = (60 if mode == "full" else 10**9), 2
    g = ProcessGroup(workers=world, max_rounds=4096)
    ctrl = g.control
    counter, exited = AtomicCounter(0), AtomicCounter(0)

    def updater():
        s = 0
        while s < budget and not ctrl.stop.read():
            s = counter.read_and_inc()
            time.sleep(0.0005 * (1 + rank))  # ranks progress at different speeds
        if exited.add(1) + 1 == U:
            ctrl.drained.add(1)

    joined, log = [], []

    def do_round(r, final, s_cur):
        joined.append((r, final))

    def on_round(r, s_cur, k_delta, unanimous):
        log.append((r, s_cur, k_delta, unanimous))

    ths = [threading.Thread(target=updater) for _ in range(U)]
    for t in ths:
        t.start()
    n = averager_loop(ctrl, workers=world, read_counter=counter.read,
                      local_drained=lambda: exited.read() == U,
                      sync_period=lambda s: 1 if s < 30 else 8, do_round=do_round,
                      on_round=on_round, stop_after=(5 if mode == "budget" else None))
    for t in ths:
        t.join()
    # final-mean gather: each rank fills its owner shard of a 103-element vector
    shards = shard_bounds(103, world)
    mean_out = torch.zeros(103)
    lo, hi = shards[rank]
    mean_out[lo:hi] = torch.arange(lo, hi, dtype=torch.float32)
    gathered = g.gather_mean(mean_out, shards)
    out_q.put((rank, n, joined, log, counter.read(), gathered.tolist()))
    g.close()
    dist.destroy_process_group()


def _run(mode):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, mode, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(30)
        assert p.exitcode == 0
    return sorted(res)


def test_group_rounds_align_and_end_on_one_unanimous_round():
    res = _run("full")
    (r0, n0, j0, l0, c0, g0), (r1, n1, j1, l1, c1, g1) = res
    assert n0 == n1 and n0 >= 2
    assert [r for r, _ in j0] == list(range(1, n0 + 1)) == [r for r, _ in j1]
    # exactly the last round is unanimous on every rank
    for log in (l0, l1):
        assert [u for *_, u in log] == [False] * (n0 - 1) + [True]
    assert c0 == c1 == 60 + 2          # claim-then-process: budget + U
    assert g0 == g1 == list(range(103))


def test_group_round_budget_stops_updaters():
    res = _run("budget")
    (_, n0, _, l0, c0, _), (_, n1, _, l1, c1, _) = res
    assert n0 == n1 and n0 >= 5
    assert l0[-1][3] and l1[-1][3]
    assert c0 < 10**6 and c1 < 10**6


def _fd_worker(rank, world, port, out_q):
    import sys
    from pathlib import Path

    sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2203_06638_b200.group import ProcessGroup
    from paper_2203_06638_b200.nvls import share_fds

    g = ProcessGroup(workers=world, max_rounds=8)
    if rank == 0:
        r1, w1 = os.pipe()
        r2, w2 = os.pipe()
        got = share_fds(g, [r1, r2])
        g.barrier()
        os.write(w1, b"stage")
        os.write(w2, b"mean")
        g.barrier()
        out_q.put((rank, "sent"))
    else:
        got = share_fds(g, None, count=2)
        g.barrier()
        g.barrier()
        out_q.put((rank, os.read(got[0], 16).decode() + "/" + os.read(got[1], 16).decode()))
    g.close()
    dist.destroy_process_group()


def test_nvls_fd_exchange_between_ranks():
    """The multicast-handle exchange of NVLS averaging (SCM_RIGHTS over a
    Unix socket, name over torch.distributed), exercised with pipe fds: the
    ranks read what rank 0 wrote into its own descriptors."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_fd_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = sorted(q.get(timeout=120) for _ in ps)
    for p in ps:
        p.join(30)
        assert p.exitcode == 0
    assert res == [(0, "sent"), (1, "stage/mean")]
