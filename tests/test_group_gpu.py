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
                                        ("mb_sgd", ("auto", "auto")), ("pl_sgd", ("auto", "auto"))])
def test_two_process_group_on_one_gpu(algo, loops):
    """("python", "auto"): rank 0 runs the Python averager, rank 1 the native
    one (lpp_averager_run) — the two implement the same protocol over the
    shared control block."""
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_rank_main, args=(r, 2, port, algo, q, loops)) for r in range(2)]
    for p in ps:
        p.start()
    res = sorted(q.get(timeout=300) for _ in ps)
    for p in ps:
        p.join(60)
        assert p.exitcode == 0
    (_, c0, r0, f0), (_, c1, r1, f1) = res
    f0, f1 = np.array(f0), np.array(f1)
    assert np.all(np.isfinite(f0))
    if algo == "lpp_sgd":
        assert c0 == [202] and c1 == [202]
        assert r0 == r1 == list(range(1, len(r0) + 1)) and len(r0) >= 2
        assert np.array_equal(f0, f1)     # both ranks gather the same final mean
    else:
        np.testing.assert_allclose(f0, f1, atol=1e-6)
