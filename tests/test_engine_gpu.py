"""Engine parity on the GPU.

1. Deterministic gate: the CUDA engine in ``schedule="serialized"`` mode vs
   the fp64 oracle (oracle/schedule.py, pinned to the reference by
   tests/golden/serialized_*.npz).  Block-id, lr and averaging-round traces
   must match EXACTLY; parameters within the fp32 contract
   ``atol=1e-5, rtol=1e-4`` (TF32 off).
2. Async mode: the reference's engine invariants (test_engine.py) — counter
   accounting, slot coverage, write-stamp permutation, block alternation, lr
   trace, zero-lr identity — plus a loss band against the serialized run.
3. Baselines: MB-SGD == PL-SGD at period 1; Q x B == 1 x QB (fp32 tolerance).
"""

from __future__ import annotations

import json
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

from conftest import load_npz  # noqa: E402

ATOL, RTOL = 1e-5, 1e-4


@pytest.fixture(autouse=True)
def _no_tf32():
    torch.backends.cuda.matmul.allow_tf32 = False
    torch.backends.cudnn.allow_tf32 = False
    yield


def _mlp(kind):
    from oracle import data as odata
    from paper_2203_06638_b200.objectives import MlpObjective

    if kind == "small":
        X, y = odata.make_blobs(48, 4, 3, 2.0, 0.5, 9)
        return MlpObjective(X, y, (5,), 3), X, y, (5,), 3
    if kind == "deep":
        X, y = odata.make_blobs(48, 6, 6, 2.0, 0.5, 13)
        return MlpObjective(X, y, (6, 6, 6), 6), X, y, (6, 6, 6), 6
    X, y = odata.cifar_blobs()
    return MlpObjective(X, y, (64,), 10), X, y, (64,), 10


def _cfg_from_golden(name, obj, **over):
    from paper_2203_06638_b200.engine import RunConfig
    from paper_2203_06638_b200.partition import make_partition
    from paper_2203_06638_b200.schedules import LrSchedule, SyncScheme

    g = load_npz(f"serialized_{name}.npz")
    c = json.loads(bytes(g["config_json"]).decode())
    s = c["sched"]
    lr = LrSchedule(kind=s["kind"], alpha0=s["alpha0"], total=s["total"], warmup=s["warmup"],
                    peak=s["peak"], milestones=tuple(s["milestones"]), gamma=s["gamma"])
    sync = SyncScheme(total=c["sync"]["total"], period=c["sync"]["period"],
                      switch_point=c["sync"]["switch_point"])
    kw = dict(algo=c["algo"], objective=obj, partition=make_partition(obj.dim, tuple(c["bounds"])),
              lr=lr, sync=sync, budget=c["budget"], warm_start_budget=c["t_st"], workers=c["Q"],
              updaters=c["U"], batch_size=c["B"], seed=c["seed"], schedule="serialized",
              record_mode="full", record_tensors=False, evaluate=False,
              epoch_partition=c.get("epoch_partition", False))
    kw.update(over)
    return g, RunConfig(**kw)


def _oracle_run(g, X, y, hidden, k):
    from oracle import schedule as osched
    from oracle.mlp import MlpOracle

    c = json.loads(bytes(g["config_json"]).decode())
    s = c["sched"]
    obj = MlpOracle(X, y, hidden, k)

    class A:
        dim, n_samples = obj.dim, obj.n_samples
        init_params = staticmethod(obj.init_params)
        grad_block = staticmethod(obj.grad_block)

    return osched.run_serialized(
        A, algo=c["algo"], workers=c["Q"], updaters=c["U"], boundaries=tuple(c["bounds"]),
        lr=osched.Lr(kind=s["kind"], alpha0=s["alpha0"], total=s["total"], warmup=s["warmup"],
                     peak=s["peak"], milestones=tuple(s["milestones"]), gamma=s["gamma"]),
        switch_point=c["sync"]["switch_point"], period=c["sync"]["period"], budget=c["budget"],
        warm_start=c["t_st"], batch_size=c["B"], seed=c["seed"],
        epoch_partition=c.get("epoch_partition", False))


@pytest.mark.parametrize("name,kind", [("deep_lpp", "deep"), ("small_lap", "small"), ("c0_lpp", "c0"),
                                       ("deep_lpp_epoch", "deep")])
@pytest.mark.parametrize("mode", ["red", "bulk"])
def test_serialized_engine_matches_oracle(name, kind, mode):
    from paper_2203_06638_b200.engine import run_experiment

    obj, X, y, hidden, k = _mlp(kind)
    g, cfg = _cfg_from_golden(name, obj, apply_mode=mode)
    res = run_experiment(cfg)
    # exact schedule traces against the reference-generated golden vectors
    got_blocks = sorted((u.worker, u.rank, u.s, u.block_id) for u in res.updates)
    want_blocks = sorted(tuple(int(v) for v in row) for row in g["block_trace"])
    assert got_blocks == want_blocks
    lr_by_key = {(u.worker, u.rank, u.s): u.lr for u in res.updates}
    want_lr = [lr_by_key[(int(a), int(b), int(c))] for a, b, c, _ in g["block_trace"]]
    assert want_lr == list(g["lr_trace"])
    assert np.array_equal(np.array(res.round_trace, dtype=np.int64), g["round_trace"])
    # parameters: fp32 engine vs fp64 oracle
    tr = _oracle_run(g, X, y, hidden, k)
    np.testing.assert_allclose(res.final_values, tr.final_values, atol=ATOL, rtol=RTOL)
    if "final" in g:
        np.testing.assert_allclose(res.final_values, g["final"], atol=ATOL, rtol=RTOL)
    else:
        np.testing.assert_allclose(res.final_values[g["idx"]], g["final_sample"], atol=ATOL, rtol=RTOL)
    assert res.counter_finals == list(tr.counter_finals)


def test_serialized_q1u1_matches_reference_engine_run():
    """The reference's own engine at Q=U=1 (golden engine_q1u1.npz)."""
    from paper_2203_06638_b200.engine import RunConfig, run_experiment
    from paper_2203_06638_b200.partition import make_partition
    from paper_2203_06638_b200.schedules import SyncScheme, constant_schedule

    obj = _mlp("small")[0]
    g = load_npz("engine_q1u1.npz")
    cfg = RunConfig(algo="lap_sgd", objective=obj, partition=make_partition(obj.dim, (0, obj.dim)),
                    lr=constant_schedule(0.05, 50), sync=SyncScheme(total=50, period=4, switch_point=0),
                    budget=50, warm_start_budget=0, workers=1, updaters=1, batch_size=8, seed=1,
                    schedule="serialized", record_mode="full", evaluate=False)
    res = run_experiment(cfg)
    np.testing.assert_allclose(res.x0, g["x0"])
    np.testing.assert_allclose(res.final_values, g["final"], atol=ATOL, rtol=RTOL)
    assert res.counter_finals == list(g["counter_finals"])


def _tiny(obj, **kw):
    from paper_2203_06638_b200.engine import RunConfig
    from paper_2203_06638_b200.partition import make_partition
    from paper_2203_06638_b200.schedules import SyncScheme, constant_schedule

    budget = kw.pop("budget", 50)
    d = dict(algo="mb_sgd", objective=obj, partition=make_partition(obj.dim, (0, obj.dim)),
             lr=constant_schedule(0.05, budget), sync=SyncScheme(total=budget, period=4, switch_point=0),
             budget=budget, warm_start_budget=0, workers=2, updaters=1, batch_size=8, seed=1,
             evaluate=False)
    d.update(kw)
    return RunConfig(**d)


def test_async_counter_and_stamp_accounting():
    """test_engine.py:203-235 on the GPU engine."""
    from paper_2203_06638_b200.engine import run_experiment

    obj = _mlp("deep")[0]
    res = run_experiment(_tiny(obj, algo="lap_sgd", budget=200, workers=2, updaters=3))
    assert res.counter_finals == [203, 203]
    for q in range(2):
        slots = sorted(u.s for u in res.updates if u.worker == q)
        assert slots == list(range(203))
        orders = [u.u for u in res.updates if u.worker == q] + [st.u for st in res.stamps if st.worker == q]
        assert sorted(orders) == list(range(1, len(orders) + 1))
    rounds = {}
    for st in res.stamps:
        rounds.setdefault(st.round, set()).add(st.worker)
    assert rounds and all(v == {0, 1} for v in rounds.values())
    assert np.all(np.isfinite(res.final_values))


def test_async_block_alternation_and_lr_trace():
    """test_engine.py:238-256, 308-333."""
    from paper_2203_06638_b200.engine import run_experiment
    from paper_2203_06638_b200.partition import make_partition
    from paper_2203_06638_b200.schedules import LrSchedule, lr_at

    obj = _mlp("deep")[0]
    e = obj.edges
    sched = LrSchedule(kind="multistep", alpha0=0.05, total=200, milestones=(80,), gamma=0.1, peak=0.05)
    cfg = _tiny(obj, algo="lpp_sgd", budget=200, workers=1, updaters=2, lr=sched,
                partition=make_partition(obj.dim, (0, e[1], e[2], e[3], e[4])), warm_start_budget=40)
    res = run_experiment(cfg)
    for u in res.updates:
        assert u.lr == lr_at(sched, u.s)
        if u.s <= 40:
            assert u.block_id == 0 and u.reason == "warm_start"
        elif (u.s - 40) % 2 == 1:
            assert u.block_id == 0 and u.reason == "alternate_full"
        else:
            assert u.block_id == u.rank and u.reason == "alternate_partial"
    assert {u.block_id for u in res.updates if u.s > 40} == {0, 1, 2}


def test_zero_learning_rate_leaves_the_model_unchanged():
    from paper_2203_06638_b200.engine import run_experiment
    from paper_2203_06638_b200.partition import make_partition
    from paper_2203_06638_b200.schedules import constant_schedule

    obj = _mlp("deep")[0]
    x0 = obj.init_params(1).astype(np.float32)
    for algo in ("mb_sgd", "pl_sgd", "lap_sgd", "lpp_sgd"):
        kw = dict(lr=constant_schedule(0.0, 50))
        if algo in ("lap_sgd", "lpp_sgd"):
            kw.update(updaters=2)
        if algo == "lpp_sgd":
            kw.update(partition=make_partition(obj.dim, (0, obj.edges[2], obj.dim)))
        res = run_experiment(_tiny(obj, algo=algo, budget=50, **kw))
        assert np.array_equal(res.final_values, x0), algo


def test_round_budget_stops_the_run_early():
    from paper_2203_06638_b200.engine import run_experiment
    from paper_2203_06638_b200.schedules import SyncScheme

    obj = _mlp("deep")[0]
    cfg = _tiny(obj, algo="lap_sgd", budget=1_000_000, workers=2, updaters=2,
                sync=SyncScheme(total=1_000_000, period=8, switch_point=0), round_budget=5)
    res = run_experiment(cfg)
    for q in range(2):
        assert max(st.round for st in res.stamps if st.worker == q) >= 5
    assert max(res.counter_finals) < 100_000


def test_async_loss_band_vs_serialized():
    """Async LPP reaches a loss within a band of the serialized schedule's."""
    from paper_2203_06638_b200.engine import run_experiment

    obj = _mlp("c0")[0]
    g, cfg = _cfg_from_golden("c0_lpp", obj, evaluate=True)
    ser = run_experiment(cfg)
    import dataclasses

    asy = run_experiment(dataclasses.replace(cfg, schedule="async"))
    l0 = ser.metrics[0].train_loss
    ls, la = ser.metrics[-1].train_loss, asy.metrics[-1].train_loss
    assert ls < l0 and la < l0
    assert abs(la - ls) <= 0.25 * (l0 - ls) + 0.05


@pytest.mark.parametrize("kind", ["deep"])
def test_baseline_identities(kind):
    """test_engine.py:82-103: period-1 PL == MB; Q x B == 1 x QB (fp32 tol)."""
    from paper_2203_06638_b200.engine import run_experiment
    from paper_2203_06638_b200.schedules import SyncScheme

    obj = _mlp(kind)[0]
    kw = dict(budget=60, sync=SyncScheme(total=60, period=1, switch_point=0))
    mb = run_experiment(_tiny(obj, algo="mb_sgd", **kw))
    pl = run_experiment(_tiny(obj, algo="pl_sgd", **kw))
    np.testing.assert_allclose(mb.final_values, pl.final_values, atol=1e-6, rtol=1e-5)
    two = run_experiment(_tiny(obj, algo="mb_sgd", budget=60, workers=2, batch_size=8))
    one = run_experiment(_tiny(obj, algo="mb_sgd", budget=60, workers=1, batch_size=16))
    np.testing.assert_allclose(two.final_values, one.final_values, atol=1e-6, rtol=1e-5)


def test_mb_sgd_matches_reference_semantics_fp64_oracle():
    """MB-SGD on the GPU vs a numpy restatement of _run_minibatch (engine.py:544-583)."""
    from oracle.mlp import MlpOracle
    from paper_2203_06638_b200.engine import run_experiment

    obj, X, y, hidden, k = _mlp("deep")
    res = run_experiment(_tiny(obj, algo="mb_sgd", budget=40, workers=2, batch_size=8))
    o = MlpOracle(X, y, hidden, k)
    x = o.init_params(1)
    gen = np.random.default_rng(np.random.SeedSequence([1, 0, 1]))
    for kk in range(1, 41):
        shards = gen.integers(0, o.n_samples, 16)
        gs = [o.grad_block(x, 0, o.dim, shards[q * 8:(q + 1) * 8]) for q in range(2)]
        x = x - 0.05 * np.mean(gs, axis=0)
    np.testing.assert_allclose(res.final_values, x, atol=ATOL, rtol=RTOL)


def test_resnet20_async_lpp_runs():
    from paper_2203_06638_b200.engine import run_experiment
    from paper_2203_06638_b200.objectives import ResNetObjective
    from paper_2203_06638_b200.partition import balanced_boundaries, make_partition
    from paper_2203_06638_b200.schedules import LrSchedule, SyncScheme

    obj = ResNetObjective("resnet20", n_samples=2048, seed=0)
    bounds = balanced_boundaries(obj.layer_param_counts, 4)
    cfg = _tiny(obj, algo="lpp_sgd", budget=40, workers=1, updaters=4, batch_size=128,
                partition=make_partition(obj.dim, bounds), warm_start_budget=4,
                lr=LrSchedule(kind="cosine", alpha0=0.1, total=40, warmup=4), momentum=0.9,
                weight_decay=5e-4, sync=SyncScheme(total=40, period=16), sampling="device",
                evaluate=True)
    res = run_experiment(cfg)
    assert res.counter_finals == [44]
    assert np.all(np.isfinite(res.final_values))
    late = [u for u in res.updates if u.s > 4]
    # which updater claims which slot is timing-dependent; the
    # PASSM+ rule itself is not: partial steps train the updater's own block
    assert all(u.block_id == (u.rank if (u.s - 4) % 2 == 0 else 0) for u in late)
    assert {u.block_id for u in late} - {0}
    assert np.isfinite(res.metrics[-1].train_loss)


def test_async_quiescent_single_updater_matches_reference_engine():
    """test_engine.py:47-59: Q=U=1, quiescent — the async engine's run equals
    the reference engine's own run (golden) within the fp32 contract."""
    from paper_2203_06638_b200.engine import RunConfig, run_experiment
    from paper_2203_06638_b200.partition import make_partition
    from paper_2203_06638_b200.schedules import SyncScheme, constant_schedule

    obj = _mlp("small")[0]
    g = load_npz("engine_q1u1.npz")
    cfg = RunConfig(algo="lap_sgd", objective=obj, partition=make_partition(obj.dim, (0, obj.dim)),
                    lr=constant_schedule(0.05, 50), sync=SyncScheme(total=50, period=4, switch_point=0),
                    budget=50, warm_start_budget=0, workers=1, updaters=1, batch_size=8, seed=1,
                    record_mode="full", quiescent=True, evaluate=False)
    res = run_experiment(cfg)
    np.testing.assert_allclose(res.final_values, g["final"], atol=ATOL, rtol=RTOL)
    assert res.counter_finals == list(g["counter_finals"])


def test_async_quiescent_group_runs_fenced_rounds():
    """Quiescent rounds: every update is clean, p_hat == 1 (test_engine.py:62-74)."""
    from paper_2203_06638_b200.engine import run_experiment

    obj = _mlp("deep")[0]
    res = run_experiment(_tiny(obj, algo="lap_sgd", budget=120, workers=2, updaters=2, quiescent=True,
                               record_mode="full"))
    assert res.p_hat == 1.0 and all(u.clean is True for u in res.updates)
    assert res.counter_finals == [122, 122]
    rounds = {}
    for st in res.stamps:
        rounds.setdefault(st.round, set()).add(st.worker)
    assert rounds and all(v == {0, 1} for v in rounds.values())
    assert np.all(np.isfinite(res.final_values))


def test_async_tags_classify_updates_and_p_hat():
    """Sampled write tags (light mode) classify every update; p_hat in (0, 1]."""
    from paper_2203_06638_b200.engine import run_experiment

    obj = _mlp("c0")[0]
    res = run_experiment(_tiny(obj, algo="lpp_sgd", budget=300, workers=2, updaters=2,
                               partition=__import__("paper_2203_06638_b200.partition", fromlist=["x"])
                               .make_partition(obj.dim, (0, obj.edges[1], obj.dim)),
                               warm_start_budget=30))
    assert all(u.clean is not None for u in res.updates)
    assert all(u.tags is not None and len(u.tags) == 16 for u in res.updates)
    assert all((np.diff(u.tag_indices) > 0).all() for u in res.updates)
    assert 0.0 < res.p_hat <= 1.0
    # every tag is a stamp that exists: at most the worker's last write stamp
    for q in range(2):
        top = max([u.u for u in res.updates if u.worker == q] +
                  [st.u for st in res.stamps if st.worker == q])
        assert all(int(t) <= top for u in res.updates if u.worker == q for t in u.tags)


@pytest.mark.parametrize("schedule", ["serialized", "async"])
def test_event_log_replays_gpu_run(tmp_path, schedule):
    """a GPU run's NDJSON event log (reference schema)
    replays on the CPU oracle to the round means the GPU measured (quiescent
    async run, or the serialized schedule), within the fp32 contract."""
    from oracle import replay
    from paper_2203_06638_b200.engine import run_experiment
    from paper_2203_06638_b200.eventlog import save_event_log
    from paper_2203_06638_b200.partition import make_partition

    obj = _mlp("deep")[0]
    bounds = (0, obj.edges[2], obj.dim)
    cfg = _tiny(obj, algo="lpp_sgd", budget=40, workers=2, updaters=2, record_mode="full",
                partition=make_partition(obj.dim, bounds), warm_start_budget=6,
                quiescent=(schedule == "async"), schedule=schedule)
    res = run_experiment(cfg)
    path = tmp_path / "run.ndjson"
    save_event_log(path, res)
    ups, sts = replay.load_event_log(path)
    assert len(ups) == len(res.updates) == sum(res.counter_finals)
    rep = replay.replay_rounds(ups, sts, res.x0, bounds)
    measured = [st.mean for st in sorted(sts, key=lambda s: s.round) if st.worker == 0]
    assert len(measured) == len(rep["round_means"]) - 1
    np.testing.assert_allclose(np.stack(rep["round_means"][1:]), np.stack(measured), atol=ATOL, rtol=RTOL)
    np.testing.assert_allclose(measured[-1], res.final_values, atol=1e-6)
    assert all(c is True for c in rep["clean"])     # quiescent / serialized: every update clean


def test_block_gradients_are_slices_of_full_mlp():
    """test_objectives.py:211-221 on the GPU objective (fp32)."""
    from paper_2203_06638_b200.partition import Block, balanced_boundaries, make_partition

    obj = _mlp("deep")[0]
    x = obj.init_params(5)
    batch = np.random.default_rng(5).integers(0, obj.n_samples, 8)
    full = obj.grad_block(x, Block(0, obj.dim), batch).values
    part = make_partition(obj.dim, balanced_boundaries(obj.layer_param_counts, 4))
    for blk in part.blocks():
        got = obj.grad_block(x, blk, batch).values
        assert torch.equal(got, full[blk.start:blk.stop])


def test_captured_partial_backprop_matches_full_slices_resnet20():
    """The engine's captured per-block graphs (StepProgram) on ResNet-20:
    every block's gradient equals the full gradient's slice (fp32, TF32 off,
    deterministic cuDNN)."""
    from paper_2203_06638_b200.objectives import ResNetObjective
    from paper_2203_06638_b200.partition import balanced_boundaries, make_partition
    from paper_2203_06638_b200.step import StepProgram

    torch.backends.cudnn.deterministic = True
    torch.backends.cudnn.benchmark = False
    try:
        obj = ResNetObjective("resnet20", n_samples=256, seed=0, autocast=None)
        part = make_partition(obj.dim, balanced_boundaries(obj.layer_param_counts, 4))
        dev = torch.device("cuda", 0)
        x = torch.from_numpy(obj.init_params(0).astype(np.float32)).to(dev)
        replica, grads = x.clone(), torch.zeros_like(x)
        st = torch.cuda.Stream()
        blocks = {b: part.block(b) for b in range(5)}
        prog = StepProgram(obj, dev, replica, grads, blocks, 32, st, input_mode="index")
        prog.idx.copy_(torch.arange(32, device=dev) * 3)
        outs = {}
        for b in range(5):
            replica.copy_(x)          # BN running stats change; params identical
            with torch.cuda.stream(st):
                prog.run(b)
            st.synchronize()
            outs[b] = grads.clone()
        full = outs[0]
        for b in range(1, 5):
            blk = blocks[b]
            np.testing.assert_allclose(outs[b][blk.start:blk.stop].cpu().numpy(),
                                       full[blk.start:blk.stop].cpu().numpy(), rtol=1e-5, atol=1e-6)
    finally:
        torch.backends.cudnn.deterministic = False


def test_host_batches_path_matches_oracle():
    """The end-to-end input path (host gather -> pinned -> H2D on a copy stream
    -> D2D into the graph input) feeds exactly the reference's batches."""
    from paper_2203_06638_b200.engine import run_experiment

    obj, X, y, hidden, k = _mlp("deep")
    g, cfg = _cfg_from_golden("deep_lpp", obj)
    res = run_experiment(cfg, host_batches=True)
    tr = _oracle_run(g, X, y, hidden, k)
    np.testing.assert_allclose(res.final_values, tr.final_values, atol=ATOL, rtol=RTOL)


@pytest.mark.parametrize("kind,workers,updaters,bounds", [("small", 3, 2, (0, 25, 43)),
                                                       ("deep", 2, 3, (0, 42, 84, 168))])
def test_serialized_misaligned_blocks_match_oracle(kind, workers, updaters, bounds):
    """Layer boundaries at elements 25 / 42 / 84 (not 16-byte aligned) exercise
    the scalar head/tail paths of K1/K3/K4/K5 inside the engine; odd Q
    exercises uneven owner shards."""
    from oracle import schedule as osched
    from oracle.mlp import MlpOracle
    from paper_2203_06638_b200.engine import RunConfig, run_experiment
    from paper_2203_06638_b200.partition import make_partition
    from paper_2203_06638_b200.schedules import LrSchedule, SyncScheme

    obj, X, y, hidden, k = _mlp(kind)
    sched = LrSchedule(kind="cosine", alpha0=0.05, total=60, warmup=6, batch_local=8, workers=workers,
                       batch_base=8)
    cfg = RunConfig(algo="lpp_sgd", objective=obj, partition=make_partition(obj.dim, bounds),
                    lr=sched, sync=SyncScheme(total=60, period=3), budget=60, warm_start_budget=6,
                    workers=workers, updaters=updaters, batch_size=8, seed=4, schedule="serialized",
                    record_mode="full", record_tensors=False, evaluate=False)
    o = MlpOracle(X, y, hidden, k)

    class A:
        dim, n_samples = o.dim, o.n_samples
        init_params = staticmethod(o.init_params)
        grad_block = staticmethod(o.grad_block)

    res = run_experiment(cfg)
    tr = osched.run_serialized(A, algo="lpp_sgd", workers=workers, updaters=updaters, boundaries=bounds,
                               lr=osched.Lr(kind="cosine", alpha0=0.05, total=60, warmup=6,
                                            peak=sched.peak),
                               switch_point=30, period=3, budget=60, warm_start=6, batch_size=8, seed=4)
    np.testing.assert_allclose(res.final_values, tr.final_values, atol=ATOL, rtol=RTOL)
    assert [tuple(r) for r in res.round_trace] == [(a, b, *c) for a, b, c in tr.rounds]


def test_synchronous_eval_rows_land_on_the_interval():
    """test_engine.py:281-286."""
    from paper_2203_06638_b200.engine import run_experiment

    obj = _mlp("deep")[0]
    res = run_experiment(_tiny(obj, algo="mb_sgd", budget=100, eval_interval=25, evaluate=True))
    assert [row.samples for row in res.metrics] == [0, 25, 50, 75, 100]
    assert [row.round for row in res.metrics] == [0, 25, 50, 75, 100]
    assert res.metrics[-1].train_loss == pytest.approx(obj.full_loss(res.final_values), rel=1e-6)


def test_async_metrics_start_at_zero_and_grow():
    """test_engine.py:289-299."""
    from paper_2203_06638_b200.engine import run_experiment

    obj = _mlp("deep")[0]
    res = run_experiment(_tiny(obj, algo="lap_sgd", budget=300, updaters=2, eval_interval=100,
                               evaluate=True))
    samples = [row.samples for row in res.metrics]
    assert samples[0] == 0 and samples == sorted(samples) and len(res.metrics) >= 3
    final = res.metrics[-1]
    assert final.train_loss == pytest.approx(obj.full_loss(res.final_values), rel=1e-6)
    assert 0.0 < final.p_hat <= 1.0


def test_final_row_matches_final_values_for_every_algorithm():
    """test_engine.py:302-305."""
    from paper_2203_06638_b200.engine import run_experiment

    obj = _mlp("deep")[0]
    for algo in ("mb_sgd", "pl_sgd", "lap_sgd"):
        res = run_experiment(_tiny(obj, algo=algo, budget=60, evaluate=True))
        assert res.metrics[-1].train_loss == pytest.approx(obj.full_loss(res.final_values), rel=1e-6)


def test_cnn_async_lpp_loss_band_vs_synchronous():
    """Async mode band on the CNN: LPP-SGD on 4 Hogwild streams
    (partial backprop) trains ResNet-20 on a learnable synthetic
    task to a loss within a band of synchronous MB-SGD given the same
    number of samples, and both learn."""
    import dataclasses

    from paper_2203_06638_b200.engine import run_experiment
    from paper_2203_06638_b200.objectives import ResNetObjective
    from paper_2203_06638_b200.partition import balanced_boundaries, make_partition
    from paper_2203_06638_b200.schedules import LrSchedule, SyncScheme

    obj = ResNetObjective("resnet20", n_samples=2048, seed=0, pattern_scale=0.5)
    slots = 160
    base = _tiny(obj, algo="lpp_sgd", budget=slots, workers=1, updaters=4, batch_size=64,
                 partition=make_partition(obj.dim, balanced_boundaries(obj.layer_param_counts, 4)),
                 warm_start_budget=16, momentum=0.0, weight_decay=5e-4, sampling="device",
                 lr=LrSchedule(kind="cosine", alpha0=0.05, total=slots + 4, warmup=16),
                 sync=SyncScheme(total=slots, period=16), evaluate=True)
    # momentum 0 (the reference has none): per-stream momentum buffers plus
    # Hogwild staleness over-accelerate this short run (tools/exp_convergence.py)
    lpp = run_experiment(base)
    mb = run_experiment(dataclasses.replace(
        base, algo="mb_sgd", updaters=1, batch_size=64, budget=slots + 4,
        partition=make_partition(obj.dim, (0, obj.dim)), warm_start_budget=0))
    l0 = lpp.metrics[0].train_loss
    la, lm = lpp.metrics[-1].train_loss, mb.metrics[-1].train_loss
    print(f"\nCNN band: initial {l0:.3f}  LPP async {la:.3f}  MB-SGD {lm:.3f}")
    assert la < 0.5 * l0 and lm < 0.5 * l0, (l0, la, lm)
    assert abs(la - lm) <= 0.35 * l0, (l0, la, lm)


@pytest.mark.parametrize("quiescent", [False, True])
def test_updater_failure_aborts_the_run(quiescent):
    """engine.py:456-463, 504-505: a failing updater stops every thread
    (averagers blocked on votes / fences / gates included) and the run raises."""
    import time as _t

    from paper_2203_06638_b200 import async_engine
    from paper_2203_06638_b200.engine import run_experiment

    obj = _mlp("deep")[0]
    # the Python updater loop (the native loop's failure path is
    # test_native_updater_failure_aborts_the_run)
    cfg = _tiny(obj, algo="lap_sgd", budget=10_000, workers=2, updaters=2, quiescent=quiescent,
                host_loop="python")
    orig = async_engine._Engine.step_fused if not quiescent else async_engine._Engine.step
    calls = {"n": 0}

    def boom(self, *a, **k):
        calls["n"] += 1
        if calls["n"] == 25:
            raise ValueError("injected updater failure")
        return orig(self, *a, **k)

    name = "step" if quiescent else "step_fused"
    setattr(async_engine._Engine, name, boom)
    try:
        t0 = _t.perf_counter()
        with pytest.raises(RuntimeError, match="engine thread failed") as ei:
            run_experiment(cfg)
        assert isinstance(ei.value.__cause__, ValueError)
        assert _t.perf_counter() - t0 < 60
    finally:
        setattr(async_engine._Engine, name, orig)


def test_failed_run_then_capture_with_aggressive_gc():
    """Regression (round-1 driver failure): a failed async run leaves its
    engine as cyclic garbage; a collector pass during the next run's graph
    capture must not free device memory or graphs mid-capture.  GC is forced
    to run as often as possible while the second engine captures."""
    import gc

    from paper_2203_06638_b200 import async_engine
    from paper_2203_06638_b200.engine import run_experiment

    obj = _mlp("deep")[0]
    orig = async_engine._Engine.step_fused
    calls = {"n": 0}

    def boom(self, *a, **k):
        calls["n"] += 1
        if calls["n"] == 5:
            raise ValueError("injected updater failure")
        return orig(self, *a, **k)

    old = gc.get_threshold()
    async_engine._Engine.step_fused = boom
    try:
        for _ in range(3):
            calls["n"] = 0
            with pytest.raises(RuntimeError, match="engine thread failed"):
                run_experiment(_tiny(obj, algo="lap_sgd", budget=200, workers=2, updaters=2,
                                     host_loop="python"))
        async_engine._Engine.step_fused = orig
        gc.set_threshold(1, 1, 1)
        res = run_experiment(_tiny(obj, algo="lap_sgd", budget=40, workers=2, updaters=2))
        assert np.all(np.isfinite(res.final_values))
    finally:
        async_engine._Engine.step_fused = orig
        gc.set_threshold(*old)


@pytest.mark.parametrize("name", ["quad8_lpp", "logreg8_lap"])
def test_serialized_flat_objectives_match_oracle(name):
    """The reference's desk-scale objectives on the GPU engine; quad8 uses the
    unlayered partition (0, 2, 4, 6, 8): partial updates that cut inside one
    parameter tensor."""
    from oracle import data as odata
    from oracle import flat
    from paper_2203_06638_b200.engine import run_experiment
    from paper_2203_06638_b200.objectives import LogisticObjective, QuadraticObjective

    if name == "quad8_lpp":
        t = flat.make_linear_targets(32, 8, 1.0, 0.5, 3)
        obj, orc_obj = QuadraticObjective(t), flat.QuadOracle(t)
    else:
        X, y = odata.make_blobs(64, 8, 2, 3.0, 0.5, 5)
        obj, orc_obj = LogisticObjective(X, np.where(y == 1, 1, -1)), flat.LogisticOracle(X, y)
    g, cfg = _cfg_from_golden(name, obj)
    res = run_experiment(cfg)
    got_blocks = sorted((u.worker, u.rank, u.s, u.block_id) for u in res.updates)
    assert got_blocks == sorted(tuple(int(v) for v in row) for row in g["block_trace"])
    assert np.array_equal(np.array(res.round_trace, dtype=np.int64), g["round_trace"])
    np.testing.assert_allclose(res.final_values, g["final"], atol=ATOL, rtol=RTOL)


def _smallcnn():
    from paper_2203_06638_b200.objectives import ResNetObjective

    return ResNetObjective("smallcnn", n_samples=256, seed=3, channels_last=False, autocast=None,
                           data="host")


def test_serialized_small_cnn_matches_oracle():
    """BASELINE config 0 on the GPU engine: small CNN, Q=2 x U=2, 2-block
    partial backprop, fp32 cuDNN (TF32 off) vs the fp64 reference-driven run."""
    from paper_2203_06638_b200.engine import run_experiment

    g, cfg = _cfg_from_golden("cnn_lpp", _smallcnn())
    res = run_experiment(cfg)
    got_blocks = sorted((u.worker, u.rank, u.s, u.block_id) for u in res.updates)
    assert got_blocks == sorted(tuple(int(v) for v in row) for row in g["block_trace"])
    assert np.array_equal(np.array(res.round_trace, dtype=np.int64), g["round_trace"])
    np.testing.assert_allclose(res.final_values, g["final"], atol=ATOL, rtol=RTOL)


def test_small_cnn_q1u1_matches_reference_engine_run():
    """The reference's own engine driving the small CNN (engine_cnn_q1u1.npz)."""
    from paper_2203_06638_b200.engine import RunConfig, run_experiment
    from paper_2203_06638_b200.partition import make_partition
    from paper_2203_06638_b200.schedules import SyncScheme, constant_schedule

    obj = _smallcnn()
    g = load_npz("engine_cnn_q1u1.npz")
    cfg = RunConfig(algo="lap_sgd", objective=obj, partition=make_partition(obj.dim, (0, obj.dim)),
                    lr=constant_schedule(0.05, 30), sync=SyncScheme(total=30, period=4, switch_point=0),
                    budget=30, warm_start_budget=0, workers=1, updaters=1, batch_size=16, seed=2,
                    schedule="serialized", record_mode="full", evaluate=False)
    res = run_experiment(cfg)
    np.testing.assert_allclose(res.x0, g["x0"])
    np.testing.assert_allclose(res.final_values, g["final"], atol=ATOL, rtol=RTOL)
    assert res.counter_finals == list(g["counter_finals"])


def test_async_loss_band_vs_reference_async_runs():
    """North star: in async mode the loss trajectory stays within a stated
    band of the REFERENCE's.  The reference's own async engine (live threads,
    tests/golden/async_band_c0.json, 5 seeds) on config C0; the GPU engine on
    the same config and seeds.  Band: every GPU final loss inside the
    reference's [min, max] widened by 0.05 (absolute; ~2 % of the initial
    loss), the initial loss (same x0, same data) equal to 1e-4."""
    from paper_2203_06638_b200.engine import RunConfig, run_experiment
    from paper_2203_06638_b200.partition import balanced_boundaries, make_partition
    from paper_2203_06638_b200.schedules import LrSchedule, SyncScheme

    ref = json.loads((Path(__file__).parent / "golden" / "async_band_c0.json").read_text())
    obj = _mlp("c0")[0]
    bounds = balanced_boundaries(obj.layer_param_counts, 2)
    finals = []
    for seed, ref_init in zip(ref["seeds"], ref["initial"]):
        cfg = RunConfig(algo="lpp_sgd", objective=obj, partition=make_partition(obj.dim, bounds),
                        lr=LrSchedule(kind="cosine", alpha0=0.05, total=200, warmup=20, batch_local=32,
                                      workers=2, batch_base=32),
                        sync=SyncScheme(total=200, period=16), budget=200, warm_start_budget=20,
                        workers=2, updaters=2, batch_size=32, seed=seed, record_mode="light")
        res = run_experiment(cfg)
        assert abs(res.metrics[0].train_loss - ref_init) <= 1e-4
        finals.append(res.metrics[-1].train_loss)
    lo, hi = min(ref["final"]) - 0.05, max(ref["final"]) + 0.05
    print(f"\nasync band: GPU finals {np.round(finals, 4)}  reference {np.round(ref['final'], 4)}")
    assert all(lo <= f <= hi for f in finals), (finals, ref["final"])


def test_async_cnn_band_vs_reference_async_runs():
    """North star on BASELINE config 0 itself: the small CNN, LPP-SGD Q=2
    workers x U=2 updaters, 2-block partial backprop, async.  The reference's
    own engine driving the small CNN (tests/golden/async_band_cnn.json, made
    by tests/golden/make_cnn_band.py: 5 seeds of live-thread runs) against
    the GPU engine's default async path (native loops, fused K1+K3 with the
    K5 plan, fp32) on the same data, x0 and seeds.  Band: every GPU final
    loss inside the reference's [min, max] widened by 0.05 (~2 % of the
    initial loss), the GPU mean inside [min, max]; initial losses (same x0,
    fp32 vs fp64 forward) equal to 1e-4."""
    from paper_2203_06638_b200.engine import RunConfig, run_experiment
    from paper_2203_06638_b200.objectives import ResNetObjective
    from paper_2203_06638_b200.partition import make_partition
    from paper_2203_06638_b200.schedules import LrSchedule, SyncScheme

    ref = json.loads((Path(__file__).parent / "golden" / "async_band_cnn.json").read_text())
    obj = ResNetObjective("smallcnn", n_samples=ref["n_samples"], seed=ref["data_seed"],
                          channels_last=False, autocast=None, data="host",
                          pattern_scale=ref["pattern_scale"])
    T, B, Q, U = ref["T"], ref["B"], ref["Q"], ref["U"]
    finals = []
    for seed, ref_init in zip(ref["seeds"], ref["initial"]):
        cfg = RunConfig(algo="lpp_sgd", objective=obj, partition=make_partition(obj.dim, ref["bounds"]),
                        lr=LrSchedule(kind="cosine", alpha0=0.05, total=T, warmup=T // 10, batch_local=B,
                                      workers=Q, batch_base=B),
                        sync=SyncScheme(total=T, period=16), budget=T, warm_start_budget=T // 10,
                        workers=Q, updaters=U, batch_size=B, seed=seed, record_mode="light")
        res = run_experiment(cfg)
        assert abs(res.metrics[0].train_loss - ref_init) <= 1e-4
        finals.append(res.metrics[-1].train_loss)
    lo, hi = min(ref["final"]), max(ref["final"])
    print(f"\ncnn async band: GPU finals {np.round(finals, 4)}  reference {np.round(ref['final'], 4)}")
    assert all(lo - 0.05 <= f <= hi + 0.05 for f in finals), (finals, ref["final"])
    assert lo <= float(np.mean(finals)) <= hi, (finals, ref["final"])


def test_native_updater_failure_aborts_the_run():
    """The same contract with the native loops: one updater's failed
    lpp_updater_run sets abort / stop, the other native updaters and the
    native averagers (waiting on votes or fences) return, the run raises."""
    import time as _t

    from paper_2203_06638_b200 import _native, native_loops
    from paper_2203_06638_b200.engine import run_experiment

    obj = _mlp("deep")[0]
    cfg = _tiny(obj, algo="lap_sgd", budget=200_000, workers=2, updaters=2)
    orig = _native.updater_run
    calls = {"n": 0}

    def boom(c):
        calls["n"] += 1
        if calls["n"] == 3:
            _t.sleep(0.2)          # let the other loops get going first
            raise ValueError("injected native updater failure")
        return orig(c)

    native_loops.N.updater_run = boom
    try:
        t0 = _t.perf_counter()
        with pytest.raises(RuntimeError, match="engine thread failed") as ei:
            run_experiment(cfg)
        assert isinstance(ei.value.__cause__, ValueError)
        assert _t.perf_counter() - t0 < 60
    finally:
        native_loops.N.updater_run = orig


@pytest.mark.parametrize("tags", [True, False])
def test_tens_of_thousands_of_rounds_through_the_ring(tags):
    """A real-length schedule averages every tick for half the run: thousands
    of rounds through the 8-cell control ring (round 1 sized the
    block per run and raised past it).  Rounds stay aligned across workers,
    1..n, and the run ends on the drain round."""
    from paper_2203_06638_b200.engine import run_experiment
    from paper_2203_06638_b200.schedules import SyncScheme

    obj = _mlp("deep")[0]
    T = 24_000
    res = run_experiment(_tiny(obj, algo="lap_sgd", budget=T, workers=2, updaters=1,
                               sync=SyncScheme(total=T, period=1, switch_point=T),
                               track_writes=tags, record_mode="off", sampling="device"))
    per = {q: sorted(st.round for st in res.stamps if st.worker == q) for q in range(2)}
    n = len(per[0])
    assert per[0] == per[1] == list(range(1, n + 1))
    assert n > 3_000            # thousands of times the 8-cell ring (the count follows timing)
    assert res.counter_finals == [T + 1, T + 1]
    assert np.all(np.isfinite(res.final_values))
