"""One process per worker, on ONE GPU: two ranks (gloo plumbing) map each
other's arenas through CUDA IPC, share the round-control block in POSIX
shared memory and run async LPP-SGD with the owner-computes K4 over the
IPC-mapped peer arena.  No kernel waits on another rank (the rendezvous is
host-side, between averager threads), so co-locating the ranks on one
device is safe.  Checks the reference invariants end to end."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank_main(rank, world, port, algo, out_q, loops=("auto", "auto")):
    import sys
    from pathlib import Path

    sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
    sys.path.insert(0, str(Path(__file__).resolve().parent))
    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.backends.cuda.matmul.allow_tf32 = False
    from oracle import data as odata
    from paper_2203_06638_b200.engine import RunConfig, run_experiment
    from paper_2203_06638_b200.group import ProcessGroup
    from paper_2203_06638_b200.objectives import MlpObjective
    from paper_2203_06638_b200.partition import make_partition
    from paper_2203_06638_b200.schedules import SyncScheme, constant_schedule

    X, y = odata.make_blobs(48, 6, 6, 2.0, 0.5, 13)
    obj = MlpObjective(X, y, (6, 6, 6), 6)
    e = obj.edges
    budget = 200
    cfg = RunConfig(algo=algo, objective=obj,
                    partition=make_partition(obj.dim, (0, e[2], obj.dim) if algo == "lpp_sgd" else (0, obj.dim)),
                    lr=constant_schedule(0.05, budget), sync=SyncScheme(total=budget, period=4),
                    budget=budget, warm_start_budget=20, workers=world,
                    updaters=2 if algo == "lpp_sgd" else 1, batch_size=8, seed=1, evaluate=False,
                    host_loop=loops[rank])
    g = ProcessGroup(workers=world, max_rounds=4096)
    res = run_experiment(cfg, group=g)
    rounds = [st.round for st in res.stamps]
    out_q.put((rank, res.counter_finals, rounds, res.final_values.tolist()))
    g.close()
    dist.destroy_process_group()


@pytest.mark.parametrize("algo,loops", [("lpp_sgd", ("auto", "auto")), ("lpp_sgd", ("python", "auto")),
                                        ("lpp_sgd", ("auto", "python", "auto", "auto")),
                                        ("mb_sgd", ("auto", "auto")), ("pl_sgd", ("auto", "auto"))])
def test_process_group_on_one_gpu(algo, loops):
    """One process per worker (2 or 4 ranks on one GPU).  A "python" entry
    runs that rank's Python averager / updater loops, "auto" the native ones
    (lpp_averager_run) — both implement the same protocol over the shared
    control block, so mixed groups must agree."""
    import torch.multiprocessing as mp

    world = len(loops)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_rank_main, args=(r, world, port, algo, q, loops)) for r in range(world)]
    for p in ps:
        p.start()
    res = sorted(q.get(timeout=300) for _ in ps)
    for p in ps:
        p.join(60)
        assert p.exitcode == 0
    counters = [c for _, c, _, _ in res]
    rounds = [r for _, _, r, _ in res]
    finals = [np.array(f) for _, _, _, f in res]
    assert np.all(np.isfinite(finals[0]))
    if algo == "lpp_sgd":
        assert all(c == [202] for c in counters)
        assert all(r == rounds[0] for r in rounds)
        assert rounds[0] == list(range(1, len(rounds[0]) + 1)) and len(rounds[0]) >= 2
        for f in finals[1:]:
            assert np.array_equal(f, finals[0])     # every rank gathers the same final mean
    else:
        for f in finals[1:]:
            np.testing.assert_allclose(f, finals[0], atol=1e-6)
