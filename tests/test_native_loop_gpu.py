"""The native updater loop (lpp_updater_run, a10 in C++) and the in-graph
device sampler, on the GPU.

The loop must keep the reference engine's updater contract
(test_engine.py:203-235): claim-then-process (each updater processes
exactly one slot >= budget, so counter_final = budget + U), every step's
flops accounted, sampled write tags classified once per step; and it must
train like the Python loop it replaces (same kernels, same sampler).
"""

from __future__ import annotations

import dataclasses

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _resnet_cfg(obj, budget=40, workers=1, updaters=4, **kw):
    from paper_2203_06638_b200.engine import RunConfig
    from paper_2203_06638_b200.partition import balanced_boundaries, make_partition
    from paper_2203_06638_b200.schedules import LrSchedule, SyncScheme

    d = dict(algo="lpp_sgd", objective=obj,
             partition=make_partition(obj.dim, balanced_boundaries(obj.layer_param_counts, updaters)),
             lr=LrSchedule(kind="cosine", alpha0=0.05, total=budget + 4, warmup=4),
             sync=SyncScheme(total=budget, period=8), budget=budget, warm_start_budget=4,
             workers=workers, updaters=updaters, batch_size=64, seed=1, momentum=0.9,
             weight_decay=5e-4, sampling="device", record_mode="off", evaluate=False,
             host_loop="native")
    d.update(kw)
    return RunConfig(**d)


def test_device_sampler_matches_host_twin_and_advances_in_graph():
    from paper_2203_06638_b200 import _native as N

    idx = torch.zeros(100, dtype=torch.long, device="cuda")
    step = torch.zeros(1, dtype=torch.long, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    for t in range(3):
        N.sample_indices(idx.data_ptr(), step.data_ptr(), 100, 5000, 42, st)
        torch.cuda.synchronize()
        assert np.array_equal(idx.cpu().numpy(), N.sample_indices_host(100, 5000, 42, t))
    assert int(step) == 3
    # captured once, every replay draws the next step's batch
    s = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        N.sample_indices(idx.data_ptr(), step.data_ptr(), 100, 5000, 42, s.cuda_stream)
    torch.cuda.synchronize()
    start = int(step)
    for t in range(start, start + 3):
        g.replay()
        torch.cuda.synchronize()
        assert np.array_equal(idx.cpu().numpy(), N.sample_indices_host(100, 5000, 42, t))


@pytest.mark.parametrize("fuse,tags", [(True, True), (False, True), (True, False), (False, False)])
def test_native_loop_accounting(fuse, tags):
    from paper_2203_06638_b200.engine import Trainer
    from paper_2203_06638_b200.objectives import ResNetObjective

    obj = ResNetObjective("resnet20", n_samples=1024, seed=0)
    cfg = _resnet_cfg(obj, budget=40, workers=2, updaters=4, fuse_snapshot=fuse, track_writes=tags)
    tr = Trainer(cfg, time_apply=True)
    try:
        assert tr.eng.native_loop()
        res = tr.run()
        assert res.counter_finals == [44, 44]          # budget + U per worker
        assert np.all(np.isfinite(res.final_values))
        steps = sum(res.counter_finals)
        n, ms, nbytes = res.apply_timing
        assert n == steps and ms > 0 and nbytes > 0
        if tags:
            assert tr.eng.classified_count.read() == steps
            assert 0.0 <= res.p_hat <= 1.0
        else:
            assert tr.eng.classified_count.read() == 0
        # flops: warm-up slots run block 0 (full); afterwards half the slots
        # are partial blocks, so the total sits strictly between the bounds
        full = tr.eng._flops_of[0]
        assert min(tr.eng._flops_of.values()) * steps <= res.flops <= full * steps
        assert res.flops < full * steps
        rounds = {}
        for st in res.stamps:
            rounds.setdefault(st.round, set()).add(st.worker)
        assert rounds and all(v == {0, 1} for v in rounds.values())
    finally:
        tr.close()


def test_native_loop_repeated_phases_and_ineligible_configs():
    from paper_2203_06638_b200.engine import Trainer
    from paper_2203_06638_b200.objectives import ResNetObjective

    obj = ResNetObjective("resnet20", n_samples=1024, seed=0)
    tr = Trainer(_resnet_cfg(obj, budget=400))
    try:
        for budget in (12, 20):
            res = tr.run(budget, evaluate=False)
            assert res.counter_finals == [budget + 4]
    finally:
        tr.close()
    with pytest.raises(ValueError, match="host_loop='native'"):
        Trainer(_resnet_cfg(obj, record_mode="full")).run()


def test_native_loop_trains_like_the_python_loop():
    """Async band: the native and Python updater loops (same kernels, same
    device sampler) both learn a learnable synthetic task and land within a
    band of each other."""
    from paper_2203_06638_b200.engine import run_experiment
    from paper_2203_06638_b200.objectives import ResNetObjective
    from paper_2203_06638_b200.schedules import LrSchedule

    obj = ResNetObjective("resnet20", n_samples=2048, seed=0, pattern_scale=0.5)
    base = _resnet_cfg(obj, budget=160, momentum=0.0, evaluate=True, warm_start_budget=16,
                       lr=LrSchedule(kind="cosine", alpha0=0.05, total=164, warmup=16))
    nat = run_experiment(base)
    py = run_experiment(dataclasses.replace(base, host_loop="python"))
    l0 = nat.metrics[0].train_loss
    ln, lp = nat.metrics[-1].train_loss, py.metrics[-1].train_loss
    print(f"\nnative {ln:.3f}  python {lp:.3f}  initial {l0:.3f}")
    assert ln < 0.5 * l0 and lp < 0.5 * l0
    assert abs(ln - lp) <= 0.25 * l0


def test_native_loop_mlp_and_lap():
    """The loop on the reference MLP objective, lap_sgd (always block 0)."""
    from paper_2203_06638_b200.engine import RunConfig, Trainer
    from paper_2203_06638_b200.objectives import MlpObjective
    from paper_2203_06638_b200.partition import make_partition
    from paper_2203_06638_b200.schedules import SyncScheme, constant_schedule

    rng = np.random.default_rng(0)
    X = rng.normal(size=(512, 32))
    y = rng.integers(0, 4, 512)
    obj = MlpObjective(X, y, (16,), 4)
    cfg = RunConfig(algo="lap_sgd", objective=obj, partition=make_partition(obj.dim, (0, obj.dim)),
                    lr=constant_schedule(0.05, 300), sync=SyncScheme(total=300, period=4),
                    budget=300, warm_start_budget=0, workers=2, updaters=3, batch_size=16, seed=3,
                    sampling="device", record_mode="off", evaluate=True, host_loop="native")
    tr = Trainer(cfg)
    try:
        res = tr.run()
        assert res.counter_finals == [303, 303]
        assert res.metrics[-1].train_loss < res.metrics[0].train_loss
    finally:
        tr.close()


@pytest.mark.parametrize("tags,workers", [(True, 2), (False, 2), (True, 3)])
def test_native_averager_round_protocol(tags, workers):
    """lpp_averager_run keeps the reference's averager contract
    (test_engine.py:152-235): every round is joined by every worker, rounds
    are numbered 1..n on both, the run ends on the drain round, the final
    values are the last round's mean — which every arena holds once all
    updaters have exited — and round stamps interleave with update stamps
    as one permutation per worker."""
    from paper_2203_06638_b200.engine import Trainer
    from paper_2203_06638_b200.objectives import ResNetObjective
    from paper_2203_06638_b200.schedules import SyncScheme

    obj = ResNetObjective("resnet20", n_samples=1024, seed=0)
    cfg = _resnet_cfg(obj, budget=60, workers=workers, updaters=3, track_writes=tags,
                      sync=SyncScheme(total=60, period=4, switch_point=10))
    tr = Trainer(cfg)
    try:
        assert tr.eng.native_averager() and tr.eng.native_loop()
        res = tr.run()
        per = {q: sorted(st.round for st in res.stamps if st.worker == q) for q in range(workers)}
        assert all(per[q] == per[0] for q in per) and per[0] == list(range(1, len(per[0]) + 1))
        assert len(per[0]) >= 3
        for q in range(workers):
            arena = tr.eng.workers[q].store.arena.tensor.cpu().numpy()
            np.testing.assert_allclose(arena, res.final_values, rtol=1e-6, atol=1e-6)
            # stamps: rounds and updates draw from the same update-order counter
            n_updates = res.counter_finals[q]
            rounds_u = sorted(st.u for st in res.stamps if st.worker == q)
            assert len(set(rounds_u)) == len(rounds_u)
            assert max(rounds_u) <= n_updates + len(rounds_u)
        if tags:
            # K5 without per-element round writes: every round publishes its
            # stamp to the worker's device round cell (the floor each
            # element's tag is raised to, add_assign's stamp, engine.py:421)
            # before the host cell; updates raise their block's stamp
            for q in range(workers):
                w = tr.eng.workers[q]
                last_u = max(st.u for st in res.stamps if st.worker == q)
                assert w.last_avg_stamp.read() == last_u
                if w.round_cell is not None:
                    assert int(w.round_cell.item()) == last_u
                assert (w.block_stamps.cpu().numpy() > 0).all()
    finally:
        tr.close()


def test_native_averager_round_budget():
    from paper_2203_06638_b200.engine import Trainer
    from paper_2203_06638_b200.objectives import ResNetObjective

    obj = ResNetObjective("resnet20", n_samples=1024, seed=0)
    tr = Trainer(_resnet_cfg(obj, budget=10_000, workers=2, updaters=2, round_budget=5))
    try:
        res = tr.run()
        assert max(st.round for st in res.stamps) >= 5      # + the drain round (engine.py:429)
        assert max(res.counter_finals) < 10_000
    finally:
        tr.close()


@pytest.mark.parametrize("fuse", [True, False])
def test_native_loop_is_bitwise_the_python_loop_without_concurrency(fuse):
    """Q = U = 1 takes the concurrency out: both loops then claim the same
    slots, draw the same in-graph batches (same sampler key and device step
    counter), compute the same lr / block and launch the same kernels — so
    the native loop's final model must equal the Python loop's bit for bit."""
    from paper_2203_06638_b200.engine import RunConfig, run_experiment
    from paper_2203_06638_b200.objectives import MlpObjective
    from paper_2203_06638_b200.partition import make_partition
    from paper_2203_06638_b200.schedules import LrSchedule, SyncScheme

    rng = np.random.default_rng(4)
    X = rng.normal(size=(256, 24))
    y = rng.integers(0, 5, 256)
    obj = MlpObjective(X, y, (12, 12), 5)
    cfg = RunConfig(algo="lpp_sgd", objective=obj,
                    partition=make_partition(obj.dim, (0, obj.edges[2], obj.dim)),
                    lr=LrSchedule(kind="cosine", alpha0=0.05, total=120, warmup=10),
                    sync=SyncScheme(total=120, period=4), budget=120, warm_start_budget=10,
                    workers=1, updaters=1, batch_size=16, seed=7, momentum=0.9, weight_decay=5e-4,
                    sampling="device", record_mode="off", evaluate=False, fuse_snapshot=fuse)
    nat = run_experiment(dataclasses.replace(cfg, host_loop="native"))
    py = run_experiment(dataclasses.replace(cfg, host_loop="python"))
    assert nat.counter_finals == py.counter_finals == [121]
    assert nat.flops == py.flops
    assert np.array_equal(nat.final_values, py.final_values)
    assert not np.array_equal(nat.final_values, nat.x0.astype(np.float32))


def test_native_loop_end_to_end_host_batches_and_loss_readback():
    """The end-to-end input path inside the native loop: host-drawn indices
    (the device sampler's stream), pinned row gather, H2D into the graphs'
    double-buffered inputs, one loss D2H per step — with the same batches
    the in-graph sampler draws, so at Q = U = 1 it trains bit for bit like
    the device-data run."""
    from paper_2203_06638_b200.engine import RunConfig, Trainer, run_experiment
    from paper_2203_06638_b200.objectives import ResNetObjective
    from paper_2203_06638_b200.partition import make_partition
    from paper_2203_06638_b200.schedules import LrSchedule, SyncScheme

    def cfg_for(obj, **kw):
        d = dict(algo="lpp_sgd", objective=obj,
                 partition=make_partition(obj.dim, (0, obj.edges[2], obj.dim)),
                 lr=LrSchedule(kind="cosine", alpha0=0.05, total=60, warmup=6),
                 sync=SyncScheme(total=60, period=4), budget=60, warm_start_budget=6, workers=1,
                 updaters=1, batch_size=32, seed=3, momentum=0.9, sampling="device",
                 record_mode="off", evaluate=False, host_loop="native")
        d.update(kw)
        return RunConfig(**d)

    host = ResNetObjective("smallcnn", n_samples=512, seed=0, data="host", channels_last=False,
                           autocast=None)
    # deterministic cuDNN algorithms so both runs do the same arithmetic
    det, bench_ = torch.backends.cudnn.deterministic, torch.backends.cudnn.benchmark
    torch.backends.cudnn.deterministic, torch.backends.cudnn.benchmark = True, False
    tr = Trainer(cfg_for(host), host_batches=True, read_loss=True)
    try:
        assert tr.eng.native_loop()
        res = tr.run()
        assert res.counter_finals == [61]
        assert len(res.losses) == 61 and np.all(np.isfinite(res.losses))
    finally:
        tr.close()
    # the same data resident on the device, batches drawn inside the graph
    try:
        ref = run_experiment(cfg_for(host))
    finally:
        torch.backends.cudnn.deterministic, torch.backends.cudnn.benchmark = det, bench_
    np.testing.assert_array_equal(res.final_values, ref.final_values)
    # and the multi-updater e2e run keeps the counter contract
    tr = Trainer(cfg_for(host, updaters=2, partition=make_partition(host.dim, (0, host.edges[2], host.edges[4], host.dim)),
                         workers=2), host_batches=True, read_loss=True)
    try:
        res = tr.run()
        assert res.counter_finals == [62, 62] and len(res.losses) == 124
    finally:
        tr.close()


def test_device_epoch_sampler_and_engine_run():
    """The epoch-partition walk on the device equals its host twin (and
    advances per replay); an async run with epoch_partition on device
    sampling keeps the counter contract through the native loop, device-
    resident and end to end."""
    from paper_2203_06638_b200 import _native as N
    from paper_2203_06638_b200.engine import Trainer
    from paper_2203_06638_b200.objectives import ResNetObjective

    idx = torch.zeros(128, dtype=torch.long, device="cuda")
    step = torch.zeros(1, dtype=torch.long, device="cuda")
    for t in range(5):
        N.sample_epoch(idx.data_ptr(), step.data_ptr(), 128, 1, 2, 25_000, 11, 0)
        torch.cuda.synchronize()
        assert np.array_equal(idx.cpu().numpy(), N.sample_epoch_host(128, 1, 2, 25_000, 11, t))
    for data, hb in (("device", False), ("host", True)):
        obj = ResNetObjective("resnet20", n_samples=1000, seed=0, data=data)
        tr = Trainer(_resnet_cfg(obj, budget=40, workers=2, updaters=2, epoch_partition=True),
                     host_batches=hb, read_loss=hb)
        try:
            assert tr.eng.native_loop()
            assert tr.eng.workers[1].programs[0].epoch == (1, 2, 500)
            res = tr.run()
            assert res.counter_finals == [42, 42] and np.all(np.isfinite(res.final_values))
        finally:
            tr.close()


def test_native_loop_light_records_keep_the_reference_invariants():
    """record_mode="light" through the native loop: one UpdateRecord per
    processed slot with the reference's invariants (test_engine.py:203-235,
    308-333) — slots 0..budget+U-1 per worker, update stamps and round
    stamps one permutation, PASSM+ block rule and reason, lr = lr_at(s),
    clean flags consistent with p_hat and with the recorded tags."""
    from paper_2203_06638_b200.engine import Trainer
    from paper_2203_06638_b200.objectives import ResNetObjective
    from paper_2203_06638_b200.schedules import lr_at

    obj = ResNetObjective("resnet20", n_samples=1024, seed=0)
    cfg = _resnet_cfg(obj, budget=60, workers=2, updaters=3, record_mode="light")
    tr = Trainer(cfg)
    try:
        assert tr.eng.native_loop()
        res = tr.run()
    finally:
        tr.close()
    assert res.counter_finals == [63, 63]
    for q in range(2):
        recs = [u for u in res.updates if u.worker == q]
        assert sorted(u.s for u in recs) == list(range(63))
        orders = [u.u for u in recs] + [st.u for st in res.stamps if st.worker == q]
        assert sorted(orders) == list(range(1, len(orders) + 1))
        for u in recs:
            want = 0 if u.s <= 4 or (u.s - 4) % 2 else u.rank
            assert u.block_id == want
            assert u.reason == ("warm_start" if u.s <= 4 else
                                "alternate_full" if (u.s - 4) % 2 else "alternate_partial")
            assert u.lr == lr_at(cfg.lr, u.s)
            assert u.clean is not None and len(u.tags) == 16
            assert u.clean == bool((u.tags >= u.k_claim).all())
            assert np.all(np.diff(u.tag_indices) > 0)
    cleans = [u.clean for u in res.updates]
    assert abs(res.p_hat - sum(cleans) / len(cleans)) < 1e-12


@pytest.mark.parametrize("in_flight", [1, 4])
def test_native_loop_in_flight_depths(in_flight):
    """The in-flight window (events per slot, staging rings of depth
    in_flight + 2) at other depths: counters, records and losses stay whole."""
    from paper_2203_06638_b200.engine import Trainer
    from paper_2203_06638_b200.objectives import ResNetObjective

    obj = ResNetObjective("resnet20", n_samples=1024, seed=0, data="host")
    tr = Trainer(_resnet_cfg(obj, budget=30, workers=1, updaters=4, in_flight=in_flight,
                             record_mode="light"), host_batches=True, read_loss=True)
    try:
        res = tr.run()
        assert res.counter_finals == [34]
        assert len(res.updates) == 34 and len(res.losses) == 34
        assert all(u.clean is not None for u in res.updates)
        assert np.all(np.isfinite(res.losses))
    finally:
        tr.close()


def test_native_averager_eval_points():
    """Eval points through lpp_averager_run (engine.py:445-451): worker 0
    keeps the round mean at every eval interval; the rows land in order,
    past each interval, with finite losses and p_hat in [0, 1]."""
    from paper_2203_06638_b200.engine import Trainer
    from paper_2203_06638_b200.objectives import ResNetObjective

    obj = ResNetObjective("resnet20", n_samples=1024, seed=0)
    tr = Trainer(_resnet_cfg(obj, budget=120, workers=2, updaters=2, eval_interval=30,
                             evaluate=True))
    try:
        assert tr.eng.native_averager() and tr.eng.native_loop()
        res = tr.run()
    finally:
        tr.close()
    samples = [row.samples for row in res.metrics]
    assert samples[0] == 0 and samples == sorted(samples) and len(res.metrics) >= 4
    mids = res.metrics[1:-1]
    assert all(30 * (i + 1) <= row.samples for i, row in enumerate(mids))
    assert all(np.isfinite(row.train_loss) and 0.0 <= row.p_hat <= 1.0 for row in res.metrics)


@pytest.mark.parametrize("fuse,epoch", [(True, False), (False, False), (True, True)])
def test_native_loop_reproduces_the_reference_rng_stream(fuse, epoch):
    """sampling="host" (the reference's numpy stream, restated in
    csrc/nprng.cu) through the native loop: at Q = U = 1 it draws the same
    sampled tag indices and batches in the same order as the Python loop —
    so the records' stream-determined fields and the final model are
    bit-identical — with i.i.d. draws or the epoch-partition sampler, fused
    or not."""
    from paper_2203_06638_b200.engine import RunConfig, run_experiment
    from paper_2203_06638_b200.objectives import MlpObjective
    from paper_2203_06638_b200.partition import make_partition
    from paper_2203_06638_b200.schedules import LrSchedule, SyncScheme

    rng = np.random.default_rng(5)
    X = rng.normal(size=(300, 20))
    y = rng.integers(0, 4, 300)
    obj = MlpObjective(X, y, (10, 10), 4)
    cfg = RunConfig(algo="lpp_sgd", objective=obj,
                    partition=make_partition(obj.dim, (0, obj.edges[2], obj.dim)),
                    lr=LrSchedule(kind="cosine", alpha0=0.05, total=80, warmup=8),
                    sync=SyncScheme(total=80, period=4), budget=80, warm_start_budget=8,
                    workers=1, updaters=1, batch_size=16, seed=11, momentum=0.9,
                    sampling="host", record_mode="light", evaluate=False, fuse_snapshot=fuse,
                    epoch_partition=epoch)
    nat = run_experiment(dataclasses.replace(cfg, host_loop="native"))
    py = run_experiment(dataclasses.replace(cfg, host_loop="python"))
    assert nat.counter_finals == py.counter_finals == [81]
    assert np.array_equal(nat.final_values, py.final_values)
    a = sorted(nat.updates, key=lambda u: u.s)
    b = sorted(py.updates, key=lambda u: u.s)
    # slots, blocks, reasons, lr and the sampled tag indices come from the
    # stream; write stamps / clean flags depend on when the averager's
    # rounds interleave (timing), so they are not compared
    assert [(u.s, u.block_id, u.reason, u.lr) for u in a] == [(u.s, u.block_id, u.reason, u.lr) for u in b]
    for u, v in zip(a, b):
        assert np.array_equal(u.tag_indices, v.tag_indices)


def test_native_end_to_end_with_the_reference_stream_matches_python():
    """End-to-end host batches drawn from the reference's numpy stream:
    native loop (pinned gather + copy-stream H2D) and Python loop train the
    small CNN bit for bit alike at Q = U = 1 (deterministic cuDNN)."""
    from paper_2203_06638_b200.engine import RunConfig, Trainer
    from paper_2203_06638_b200.objectives import ResNetObjective
    from paper_2203_06638_b200.partition import make_partition
    from paper_2203_06638_b200.schedules import LrSchedule, SyncScheme

    obj = ResNetObjective("smallcnn", n_samples=400, seed=1, data="host", channels_last=False,
                          autocast=None)
    cfg = RunConfig(algo="lpp_sgd", objective=obj,
                    partition=make_partition(obj.dim, (0, obj.edges[2], obj.dim)),
                    lr=LrSchedule(kind="cosine", alpha0=0.05, total=40, warmup=4),
                    sync=SyncScheme(total=40, period=4), budget=40, warm_start_budget=4, workers=1,
                    updaters=1, batch_size=24, seed=2, sampling="host", record_mode="light",
                    evaluate=False)
    det, bench_ = torch.backends.cudnn.deterministic, torch.backends.cudnn.benchmark
    torch.backends.cudnn.deterministic, torch.backends.cudnn.benchmark = True, False
    out = {}
    try:
        for loop in ("native", "python"):
            tr = Trainer(dataclasses.replace(cfg, host_loop=loop), host_batches=True, read_loss=True)
            try:
                assert tr.eng.native_loop() == (loop == "native")
                out[loop] = tr.run()
            finally:
                tr.close()
    finally:
        torch.backends.cudnn.deterministic, torch.backends.cudnn.benchmark = det, bench_
    assert np.array_equal(out["native"].final_values, out["python"].final_values)
    assert out["native"].losses == out["python"].losses
