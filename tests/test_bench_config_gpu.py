"""Parity of the exact configuration bench.py times, against the oracle.

bench.py's headline run is: LPP-SGD, the native C++ updater loop
(``lpp_updater_run``), the fused K1+K3 apply-and-snapshot kernel on the
high-priority apply stream, momentum 0.9 / weight decay 5e-4, K5 write tags,
the in-graph device sampler, and (for ``e2e``) host batches with an H2D copy
and a loss read-back every step.  At Q = U = 1 that pipeline is
deterministic (one stream; the next step's snapshot is taken when this
step's apply lands — engine.py:336-362 in order; averaging a single worker
is the identity, test_engine.py:169-182), so its parameters must follow the
serialized oracle (oracle/schedule.py with per-updater momentum in the
kernels' operation order, oracle/apply_ref.c ``sgd_delta``) driven by the
device sampler's batch stream restated in oracle/devsample.py.

Tolerance (fp32 engine vs fp64 oracle, TF32 off): the SURVEY §8c contract
``atol 1e-5, rtol 1e-4`` for the reference MLP (C0) and the small CNN;
ResNet-20 (ReLU kinks make its gradient non-smooth, see the test) ``atol
3e-4, rtol 1e-3`` over three steps, losses ``rtol 1e-4``.  Block ids and
learning rates are exact.

The file name sorts before test_engine_gpu.py so a later failure cannot
hide it under ``pytest -x``.
"""

from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

MU, WD = 0.9, 5e-4


@pytest.fixture(autouse=True)
def _no_tf32():
    torch.backends.cuda.matmul.allow_tf32 = False
    torch.backends.cudnn.allow_tf32 = False
    yield


def _cfg(obj, bounds, budget, B, record_mode="off", alpha0=0.1, **over):
    """bench.build_cfg at Q = U = 1 (same schedule shapes, smaller budget)."""
    from paper_2203_06638_b200.engine import RunConfig
    from paper_2203_06638_b200.partition import make_partition
    from paper_2203_06638_b200.schedules import LrSchedule, SyncScheme

    kw = dict(algo="lpp_sgd", objective=obj, partition=make_partition(obj.dim, bounds),
              lr=LrSchedule(kind="cosine", alpha0=alpha0, total=budget, warmup=max(budget // 10, 1),
                            batch_local=B, workers=1, batch_base=B, boost=True),
              sync=SyncScheme(total=budget, period=16), budget=budget,
              warm_start_budget=max(budget // 10, 1), workers=1, updaters=1, batch_size=B, seed=0,
              momentum=MU, weight_decay=WD, sampling="device", evaluate=False,
              record_mode=record_mode, host_loop="native")
    kw.update(over)
    return RunConfig(**kw)


def _oracle(orc, cfg, bounds, record_loss=False):
    from oracle import devsample
    from oracle import schedule as osched

    n, B, seed = orc.n_samples, cfg.batch_size, cfg.seed
    s = cfg.lr
    return osched.run_serialized(
        orc, algo="lpp_sgd", workers=1, updaters=1, boundaries=tuple(bounds),
        lr=osched.Lr(kind="cosine", alpha0=s.alpha0, total=s.total, warmup=s.warmup, peak=s.peak),
        switch_point=cfg.sync.switch_point, period=cfg.sync.period, budget=cfg.budget,
        warm_start=cfg.warm_start_budget, batch_size=B, seed=seed, mu=MU, wd=WD,
        batch_fn=lambda q, r, t: devsample.iid_batch(devsample.engine_key(seed, q, r), t, B, n),
        record_loss=record_loss)


def _check_trainer_flags(tr):
    eng = tr.eng
    assert eng.native_loop(), "bench config must run the native updater loop"
    assert eng.fused(), "bench config must run the fused K1+K3 kernel"
    assert eng.apply_on_side(), "bench config applies on the high-priority stream"
    assert eng.cfg.tracks, "bench config keeps K5 write tags"


def _run(cfg, host_batches=False, read_loss=False):
    from paper_2203_06638_b200 import _native as N
    from paper_2203_06638_b200.engine import Trainer

    tr = Trainer(cfg, host_batches=host_batches, read_loss=read_loss)
    try:
        _check_trainer_flags(tr)
        l0 = N.launch_count()
        res = tr.run()
        assert N.launch_count() - l0 >= cfg.budget   # our kernels ran: >= one apply per step
        return res
    finally:
        tr.close()


def _c0():
    from oracle import data as odata
    from oracle.mlp import MlpOracle
    from paper_2203_06638_b200.objectives import MlpObjective

    X, y = odata.cifar_blobs()
    obj = MlpObjective(X, y, (64,), 10)
    orc = MlpOracle(X, y, (64,), 10)
    bounds = (0, obj.edges[1], obj.dim)        # balanced_boundaries of C0: (0, 196672, 197322)
    return obj, orc, bounds


@pytest.mark.parametrize("record_mode", ["off", "light"])
def test_bench_pipeline_matches_oracle_c0_mlp(record_mode):
    obj, orc, bounds = _c0()
    cfg = _cfg(obj, bounds, budget=160, B=32, record_mode=record_mode, alpha0=0.05)
    res = _run(cfg)
    tr = _oracle(orc, cfg, bounds)
    assert res.counter_finals == tr.counter_finals == [161]
    err = float(np.max(np.abs(res.final_values - tr.final_values)))
    np.testing.assert_allclose(res.final_values, tr.final_values, atol=1e-5, rtol=1e-4,
                               err_msg=f"max |dx| = {err:.3e}")
    # the run actually moved the model (momentum + wd + partial blocks)
    assert np.max(np.abs(tr.final_values - res.x0)) > 1e-2
    if record_mode == "light":
        got = sorted((u.worker, u.rank, u.s, u.block_id) for u in res.updates)
        assert got == sorted(tr.block_ids)
        lrs = {(u.worker, u.rank, u.s): u.lr for u in res.updates}
        assert all(lrs[(q, r, s)] == lr for q, r, s, lr in tr.lrs)
        # every update is classified (clean iff no round landed in its
        # window, engine.py:357-362; at Q = 1 rounds still stamp the tags)
        assert all(u.clean is not None for u in res.updates)
        assert 0.0 <= res.p_hat <= 1.0


def test_bench_e2e_pipeline_matches_oracle_c0_mlp():
    """The e2e leg: host batches (the device sampler's stream drawn on the
    host, pinned gather, H2D per step) and the loss read back per step."""
    obj, orc, bounds = _c0()
    cfg = _cfg(obj, bounds, budget=120, B=32, alpha0=0.05)
    res = _run(cfg, host_batches=True, read_loss=True)
    tr = _oracle(orc, cfg, bounds, record_loss=True)
    np.testing.assert_allclose(res.final_values, tr.final_values, atol=1e-5, rtol=1e-4)
    want = [l for *_, l in sorted(tr.losses)]
    assert len(res.losses) == len(want)
    np.testing.assert_allclose(res.losses, want, atol=1e-5, rtol=1e-4)


def test_bench_pipeline_matches_oracle_small_cnn():
    from oracle.cnn import SmallCnnOracle
    from paper_2203_06638_b200.objectives import ResNetObjective

    obj = ResNetObjective("smallcnn", n_samples=512, seed=3, channels_last=False, autocast=None,
                          data="host")
    orc = SmallCnnOracle(obj.features.double().numpy(), obj.labels.numpy())
    e = orc.edges
    bounds = (0, e[2], e[6])                   # 2 blocks: conv1 | conv2 + fc
    cfg = _cfg(obj, bounds, budget=100, B=32, alpha0=0.05)
    res = _run(cfg)
    tr = _oracle(orc, cfg, bounds)
    np.testing.assert_allclose(res.final_values, tr.final_values, atol=1e-5, rtol=1e-4)


def test_bench_pipeline_matches_oracle_resnet20_fp32():
    """The bench's own network (ResNet-20, channels-last arena layout, fp32
    compute — the headline precision) through the bench pipeline, 4 blocks
    from balanced_boundaries as in bench.py, vs the fp64 functional oracle.

    ResNet-20's gradient is not smooth in the parameters (ReLU kinks over
    32x32 feature maps): perturbing the stem by 1e-8 moves the fp64 gradient
    by 5e-4, so fp32-vs-fp64 trajectories separate within a few steps.  The
    check therefore covers three steps (blocks 0, 0, 1: warm_start_budget 0)
    with ``atol 3e-4, rtol 1e-3`` on the parameters, and the per-step losses
    read back by the loop (``rtol 1e-6`` at x0, ``1e-4`` after)."""
    from oracle.resnet import ResNet20Oracle
    from paper_2203_06638_b200.objectives import ResNetObjective
    from paper_2203_06638_b200.partition import balanced_boundaries

    obj = ResNetObjective("resnet20", n_samples=1024, seed=0, autocast=None, channels_last=True,
                          data="device")
    bounds = balanced_boundaries(obj.layer_param_counts, 4)
    cfg = _cfg(obj, bounds, budget=2, B=32, alpha0=0.05, warm_start_budget=0)
    res = _run(cfg, read_loss=True)
    feats = obj.features_on(torch.device("cuda", 0)).double().cpu().numpy()
    orc = ResNet20Oracle(feats, obj.labels.numpy(), res.x0, channels_last=True)
    assert orc.dim == obj.dim
    tr = _oracle(orc, cfg, bounds, record_loss=True)
    assert [b for *_, b in sorted(tr.block_ids)] == [0, 0, 1]
    err = float(np.max(np.abs(res.final_values - tr.final_values)))
    np.testing.assert_allclose(res.final_values, tr.final_values, atol=3e-4, rtol=1e-3,
                               err_msg=f"max |dx| = {err:.3e}")
    assert np.max(np.abs(tr.final_values - res.x0)) > 1e-3
    want = [l for *_, l in sorted(tr.losses)]
    # the loss at x0 is one fp32 forward; later ones inherit the kink-driven
    # parameter differences above
    np.testing.assert_allclose(res.losses[0], want[0], rtol=1e-6)
    np.testing.assert_allclose(res.losses, want, rtol=1e-4)


@pytest.mark.parametrize("record_mode", ["full", "light"])
def test_serialized_momentum_q2u2_matches_oracle(record_mode):
    """Momentum 0.9 / weight decay 5e-4 (one momentum buffer per updater
    stream) with averaging across Q = 2 workers x U = 2 updaters: the
    serialized schedule (the parity mode, unfused K3 / K1) against the
    oracle; "light" records also draw the 16 sampled tag indices from each
    updater's rng before its batch (engine.py:343-351), which shifts the
    batch stream."""
    import dataclasses

    from oracle import data as odata
    from oracle import schedule as osched
    from oracle.mlp import MlpOracle
    from paper_2203_06638_b200.engine import RunConfig, run_experiment
    from paper_2203_06638_b200.objectives import MlpObjective
    from paper_2203_06638_b200.partition import make_partition
    from paper_2203_06638_b200.schedules import LrSchedule, SyncScheme

    X, y = odata.make_blobs(48, 6, 6, 2.0, 0.5, 13)
    obj = MlpObjective(X, y, (6, 6, 6), 6)
    bounds = (0, obj.edges[2], obj.dim)
    T = 80
    sched = LrSchedule(kind="cosine", alpha0=0.05, total=T, warmup=8, batch_local=8, workers=2,
                       batch_base=8, boost=True)
    cfg = RunConfig(algo="lpp_sgd", objective=obj, partition=make_partition(obj.dim, bounds), lr=sched,
                    sync=SyncScheme(total=T, period=4), budget=T, warm_start_budget=8, workers=2,
                    updaters=2, batch_size=8, seed=3, schedule="serialized", record_mode=record_mode,
                    record_tensors=False, evaluate=False, momentum=MU, weight_decay=WD)
    res = run_experiment(cfg)
    o = MlpOracle(X, y, (6, 6, 6), 6)
    tr = osched.run_serialized(
        o, algo="lpp_sgd", workers=2, updaters=2, boundaries=bounds,
        lr=osched.Lr(kind="cosine", alpha0=0.05, total=T, warmup=8, peak=sched.peak),
        switch_point=cfg.sync.switch_point, period=4, budget=T, warm_start=8, batch_size=8, seed=3,
        mu=MU, wd=WD, tag_draw=16 if record_mode == "light" else 0)
    assert sorted((u.worker, u.rank, u.s, u.block_id) for u in res.updates) == sorted(tr.block_ids)
    assert [tuple(r) for r in res.round_trace] == [(a, b, *c) for a, b, c in tr.rounds]
    np.testing.assert_allclose(res.final_values, tr.final_values, atol=1e-5, rtol=1e-4)
    assert np.max(np.abs(tr.final_values - res.x0)) > 1e-2


def test_more_than_32_sampled_tags_take_the_unfused_path():
    """The fused K5 plan carries <= 32 sampled tags in its launch; a larger
    tag_sample runs the unfused per-element path and still classifies
    every update (engine.py:343-362)."""
    obj, orc, bounds = _c0()
    cfg = _cfg(obj, bounds, budget=40, B=32, record_mode="light", tag_sample=40)
    from paper_2203_06638_b200.engine import Trainer

    tr = Trainer(cfg)
    try:
        assert not tr.eng.fused() and tr.eng.native_loop()
        res = tr.run()
    finally:
        tr.close()
    assert all(u.clean is not None and len(u.tags) == 40 for u in res.updates)
    assert all(u.clean == bool((u.tags >= u.k_claim).all()) for u in res.updates)
    tr2 = _oracle(orc, cfg, bounds)
    np.testing.assert_allclose(res.final_values, tr2.final_values, atol=1e-5, rtol=1e-4)


def test_repeated_phases_reset_k5_state_and_keep_parity():
    """Trainer phases (bench: warm-up, then the timed phase) on the same
    arenas: every phase restarts counters, the round cell and the block
    stamps; the records of the second phase satisfy the classification rule
    and its stamps start from 1 again."""
    from paper_2203_06638_b200.engine import Trainer

    obj, orc, bounds = _c0()
    cfg = _cfg(obj, bounds, budget=200, B=32, record_mode="light")
    tr = Trainer(cfg)
    try:
        r1 = tr.run(30)
        w = tr.eng.workers[0]
        assert int(w.block_stamps.max().item()) > 0
        r2 = tr.run(30)
        us = sorted(u.u for u in r2.updates)
        assert us[0] == 1 or min(st.u for st in r2.stamps) == 1     # stamps restart each phase
        assert r2.counter_finals == [31]
        assert all(u.clean == bool((u.tags >= u.k_claim).all()) for u in r2.updates)
        assert int(w.block_stamps.max().item()) <= max(us)          # no stamp from phase 1 left
    finally:
        tr.close()
    assert r1.counter_finals == [31]
