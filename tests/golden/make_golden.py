"""Generate the golden vectors that pin oracle/ to the reference.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It builds a scratch copy of the reference package (/root/reference/pkg is
read-only) under /tmp/refbuild, imports ``asyncsgd`` from there, and writes
small fixtures next to this script.  Everything here calls the reference's
OWN functions (partition, schedules, ParamStore, MlpObjective, make_blobs,
run_experiment); the canonical serialized schedule is composed
from those primitives, independently of oracle/schedule.py.

Fixtures are committed; /root/reference is never read at test time.
"""

from __future__ import annotations

import itertools
import json
import os
import shutil
import subprocess
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REF_PKG = Path(os.environ.get("LPP_REFERENCE_PKG", "/root/reference/pkg"))
SCRATCH = Path(os.environ.get("LPP_REFERENCE_SCRATCH", "/tmp/refbuild"))


def import_reference():
    if not (SCRATCH / "src" / "asyncsgd").exists():
        if SCRATCH.exists():
            shutil.rmtree(SCRATCH)
        shutil.copytree(REF_PKG, SCRATCH)
    if not list((SCRATCH / "src" / "asyncsgd").glob("_atomics*.so")):
        subprocess.run([sys.executable, "setup.py", "build_ext", "--inplace"], cwd=SCRATCH,
                       check=True, capture_output=True)
    sys.path.insert(0, str(SCRATCH / "src"))
    import asyncsgd  # noqa: F401

    return asyncsgd


def main() -> None:
    import_reference()
    from asyncsgd import data as rdata
    from asyncsgd import engine as rengine
    from asyncsgd import objectives as robj
    from asyncsgd import partition as rpart
    from asyncsgd import schedules as rsched
    from asyncsgd.paramstore import ParamStore

    out: dict = {}

    # ---------------- partition (partition.py:62-145) ----------------
    gen = np.random.default_rng(20260)
    cases = [((4, 4, 4, 4), 2), ((4, 4, 4, 4), 3), ((10, 2, 2, 10), 2), ((1, 9, 1, 9, 1), 3),
             ((6, 5, 4, 3, 2, 1), 4), ((100, 1, 1, 1), 2), ((2, 4, 2), 2), ((2, 2, 4), 2),
             ((3, 5, 7), 1), ((2, 3, 4), 3)]
    for _ in range(150):
        n = int(gen.integers(1, 11))
        sizes = tuple(int(v) for v in gen.integers(1, 40, n))
        u = int(gen.integers(1, n + 1))
        cases.append((sizes, u))
    balanced = [[list(s), u, list(rpart.balanced_boundaries(s, u))] for s, u in cases]
    # with explicit (non-negative and signed) layer costs
    costed = []
    for _ in range(60):
        n = int(gen.integers(2, 9))
        sizes = tuple(int(v) for v in gen.integers(1, 30, n))
        u = int(gen.integers(1, n + 1))
        costs = [float(c) for c in gen.normal(size=n) * 10]
        if _ % 2 == 0:
            costs = [abs(c) for c in costs]
        costed.append([list(sizes), u, costs, list(rpart.balanced_boundaries(sizes, u, costs))])
    # the config-sized MLP split used by C0
    c0 = [list((3072 * 64 + 64, 64 * 10 + 10)), 2,
          list(rpart.balanced_boundaries((3072 * 64 + 64, 64 * 10 + 10), 2))]
    selects = []
    for t_st, nb, rank in [(100, 4, 3), (0, 2, 2), (7, 2, 1), (40, 4, 1), (2000, 4, 4)]:
        ids = [rpart.select_block(s, t_st, nb, rank).block_id for s in range(0, t_st + 60)]
        reasons = [rpart.select_block(s, t_st, nb, rank).reason.value for s in range(0, t_st + 60)]
        selects.append([t_st, nb, rank, ids, reasons])
    even = [[d, k, list(rpart.even_boundaries(d, k))] for d, k in [(10, 3), (8, 4), (7, 7), (100, 6)]]
    out["partition"] = {"balanced": balanced, "costed": costed, "c0": c0, "select": selects,
                        "even": even}

    # ---------------- schedules (schedules.py:14-95) ----------------
    scheds = {
        "cos_warm": dict(kind="cosine", alpha0=0.1, total=1000, warmup=100, batch_local=64,
                         workers=2, batch_base=32),
        "cos_boost": dict(kind="cosine", alpha0=0.05, total=300, warmup=30, batch_local=32,
                          workers=2, batch_base=32, boost=True),
        "cos_plain": dict(kind="cosine", alpha0=0.1, total=500),
        "multistep": dict(kind="multistep", alpha0=0.1, total=600, warmup=10, batch_local=128,
                          workers=4, batch_base=128, milestones=(200, 400), gamma=0.1),
        "paper_r20": dict(kind="cosine", alpha0=0.1, total=117300, warmup=1955, batch_local=128,
                          workers=2, batch_base=128, boost=True),
    }
    lr_traces = {}
    for name, kw in scheds.items():
        sc = rsched.LrSchedule(**kw)
        pts = sorted(set(list(range(0, min(kw["total"], 1200) + 5)) + [kw["total"] // 2, kw["total"], kw["total"] + 7]))
        lr_traces[name] = {"kw": {k: (list(v) if isinstance(v, tuple) else v) for k, v in kw.items()},
                           "peak": sc.peak, "s": pts, "lr": [rsched.lr_at(sc, s) for s in pts]}
    syncs = []
    for total, period, sw in [(500, 4, None), (100, 16, 0), (300, 8, 120)]:
        sc = rsched.SyncScheme(total=total, period=period, switch_point=sw)
        syncs.append([total, period, sw, sc.switch_point,
                      [rsched.sync_every(sc, s) for s in range(0, total + 3)]])
    out["schedules"] = {"lr": lr_traces, "sync": syncs}

    # ---------------- ParamStore worked examples (paramstore.py:121-136) ----------------
    st = ParamStore(np.array([1.0, 2.0, 3.0, 4.0]))
    st.sub_assign(1, np.array([-10.0, -20.0]))
    ex1 = st.values.tolist()
    st2 = ParamStore(np.array([2.0, 4.0]))
    st2.add_assign(0, np.array([-1.0, 1.0]))
    ex2 = st2.values.tolist()
    st3 = ParamStore(np.zeros(4), track_writes=True)
    st3.sub_assign(1, np.array([1.0, 1.0]), stamp=7)
    ex3 = st3.snapshot().tags.tolist()
    out["paramstore"] = {"sub_assign": ex1, "add_assign": ex2, "tags": ex3}

    # ---------------- EpochSampler (objectives.py:77-104) ----------------
    epochs = []
    for n, Q, q, rank, seed, bs in [(37, 2, 0, 1, 1, 5), (37, 2, 1, 2, 1, 7), (48, 3, 2, 1, 9, 16),
                                    (10, 1, 0, 1, 3, 4)]:
        smp = robj.EpochSampler(np.arange(n)[q::Q], seed=seed * 1000 + q * 10 + rank)
        epochs.append([n, Q, q, rank, seed, bs, [smp.next_batch(bs).tolist() for _ in range(9)]])
    out["epoch_sampler"] = epochs

    (HERE / "scalars.json").write_text(json.dumps(out, indent=None, separators=(",", ":")))

    # ---------------- datasets (data.py:34-52) ----------------
    arrays = {}
    for name, args in {"blobs_small": (48, 4, 3, 2.0, 0.5, 9), "blobs_deep": (48, 6, 6, 2.0, 0.5, 13),
                       "blobs_odd": (37, 5, 4, 1.5, 0.25, 3)}.items():
        ds = rdata.make_blobs(*args)
        arrays[f"{name}_X"] = ds.features
        arrays[f"{name}_y"] = ds.labels
    c0ds = rdata.make_blobs(2048, 3072, 10, 2.5, 0.5, 11)
    arrays["c0_rows"] = c0ds.features[[0, 1, 777, 2047]]
    arrays["c0_sum"] = np.array([c0ds.features.sum(), (c0ds.features ** 2).sum()])
    arrays["c0_y"] = c0ds.labels
    np.savez_compressed(HERE / "data.npz", **arrays)

    # ---------------- MLP objective (objectives.py:200-319) ----------------
    mlp = {}
    small = robj.MlpObjective.from_dataset(rdata.make_blobs(48, 4, 3, 2.0, 0.5, 9), hidden=(5,))
    deep = robj.MlpObjective.from_dataset(rdata.make_blobs(48, 6, 6, 2.0, 0.5, 13), hidden=(6, 6, 6))
    c0 = robj.MlpObjective.from_dataset(c0ds, hidden=(64,))
    for name, obj in (("small", small), ("deep", deep)):
        x = obj.init_params(1)
        mlp[f"{name}_x0"] = x
        batch = np.random.default_rng(5).integers(0, obj.n_samples, 8)
        mlp[f"{name}_batch"] = batch
        mlp[f"{name}_loss"] = np.array([obj.loss(x, batch), obj.full_loss(x)])
        edges = np.concatenate([[0], np.cumsum(obj.layer_param_counts)])
        mlp[f"{name}_edges"] = edges
        mlp[f"{name}_gfull"] = obj.grad_block(x, rpart.Block(0, obj.dim), batch).values
        for l in range(len(edges) - 1):
            blk = rpart.Block(int(edges[l]), int(edges[-1]))
            mlp[f"{name}_gsuffix{l}"] = obj.grad_block(x, blk, batch).values
            one = rpart.Block(int(edges[l]), int(edges[l + 1]))
            mlp[f"{name}_glayer{l}"] = obj.grad_block(x, one, batch).values
            mlp[f"{name}_cost{l}"] = np.array([obj.backward_cost(one)])
    x = c0.init_params(1)
    idx = np.random.default_rng(0).integers(0, c0.dim, 2000)
    mlp["c0_idx"] = idx
    mlp["c0_x0_sample"] = x[idx]
    mlp["c0_x0_stats"] = np.array([x.sum(), (x ** 2).sum()])
    batch = np.random.default_rng(3).integers(0, c0.n_samples, 32)
    g = c0.grad_block(x, rpart.Block(0, c0.dim), batch).values
    mlp["c0_batch"] = batch
    mlp["c0_g_sample"] = g[idx]
    mlp["c0_g_stats"] = np.array([g.sum(), (g ** 2).sum()])
    mlp["c0_loss"] = np.array([c0.loss(x, batch)])
    np.savez_compressed(HERE / "mlp.npz", **mlp)

    # ---------------- canonical serialized schedule from reference primitives ----------------
    def serialized(obj, *, algo, Q, U, bounds, sched, sync, budget, t_st, B, seed,
                   epoch_partition=False):
        part = rpart.make_partition(obj.dim, bounds)
        x0 = obj.init_params(seed)
        stores = [ParamStore(x0) for _ in range(Q)]
        rngs = [[np.random.default_rng(np.random.SeedSequence([seed, q, r])) for r in range(1, U + 1)]
                for q in range(Q)]
        active = [[True] * U for _ in range(Q)]
        samplers = ([[robj.EpochSampler(np.arange(obj.n_samples)[q::Q], seed=seed * 1000 + q * 10 + r)
                      for r in range(1, U + 1)] for q in range(Q)] if epoch_partition else None)
        s_pre = [0] * Q
        block_trace, lr_trace, round_trace = [], [], []
        sweep = 0
        mean = x0.copy()
        while True:
            for q in range(Q):
                for ri in range(U):
                    if not active[q][ri]:
                        continue
                    rank = ri + 1
                    s = stores[q].read_and_inc()
                    lr = rsched.lr_at(sched, s)
                    if algo == "lpp_sgd":
                        bid = rpart.select_block(s, t_st, part.num_blocks, rank).block_id
                    else:
                        bid = 0
                    blk = part.block(bid)
                    snap = stores[q].snapshot()
                    if samplers is not None:
                        batch = samplers[q][ri].next_batch(B)
                    else:
                        batch = robj.sample_batch(rngs[q][ri], obj.n_samples, B)
                    g = obj.grad_block(snap.values, blk, batch)
                    stores[q].sub_assign(blk.start, lr * g.values)
                    block_trace.append((q, rank, s, bid))
                    lr_trace.append(lr)
                    if s >= budget:
                        active[q][ri] = False
            sweep += 1
            drained = not any(a for row in active for a in row)
            counts = [stores[q].sample_counter.read() for q in range(Q)]
            fresh = any(counts[q] - s_pre[q] >= rsched.sync_every(sync, counts[q]) for q in range(Q))
            if fresh or drained:
                slots = np.stack([stores[q].snapshot().values for q in range(Q)])
                mean = np.mean(slots, axis=0)
                for q in range(Q):
                    stores[q].add_assign(0, mean - slots[q])
                    s_pre[q] = counts[q]
                round_trace.append((len(round_trace) + 1, sweep, *counts))
            if drained:
                break
        return mean, [st.values.copy() for st in stores], block_trace, lr_trace, round_trace

    def save_serialized(name, obj, full_values, **kw):
        mean, xs, bt, lt, rt = serialized(obj, **kw)
        arr = {"block_trace": np.array(bt, dtype=np.int64), "lr_trace": np.array(lt),
               "round_trace": np.array(rt, dtype=np.int64)}
        if full_values:
            arr["final"] = mean
            arr["xs"] = np.stack(xs)
        else:
            idx = np.random.default_rng(1).integers(0, obj.dim, 4000)
            arr["idx"] = idx
            arr["final_sample"] = mean[idx]
            arr["final_stats"] = np.array([mean.sum(), (mean ** 2).sum()])
            arr["xs_sample"] = np.stack([x[idx] for x in xs])
        cfg = {k: (list(v) if isinstance(v, tuple) else v) for k, v in kw.items()
               if k not in ("sched", "sync")}
        s = kw["sched"]
        cfg["sched"] = dict(kind=s.kind, alpha0=s.alpha0, total=s.total, warmup=s.warmup,
                            peak=s.peak, milestones=list(s.milestones), gamma=s.gamma)
        cfg["sync"] = dict(total=kw["sync"].total, period=kw["sync"].period,
                           switch_point=kw["sync"].switch_point)
        arr["config_json"] = np.frombuffer(json.dumps(cfg).encode(), dtype=np.uint8)
        np.savez_compressed(HERE / f"serialized_{name}.npz", **arr)

    e = np.concatenate([[0], np.cumsum(deep.layer_param_counts)])
    save_serialized(
        "deep_lpp", deep, True, algo="lpp_sgd", Q=2, U=2, bounds=(0, int(e[2]), deep.dim),
        sched=rsched.LrSchedule(kind="cosine", alpha0=0.05, total=60, warmup=6, batch_local=8,
                                workers=2, batch_base=8, boost=True),
        sync=rsched.SyncScheme(total=60, period=4), budget=60, t_st=6, B=8, seed=1)
    e2 = np.concatenate([[0], np.cumsum(small.layer_param_counts)])
    save_serialized(
        "small_lap", small, True, algo="lap_sgd", Q=3, U=2, bounds=(0, small.dim),
        sched=rsched.constant_schedule(0.05, 40), sync=rsched.SyncScheme(total=40, period=3, switch_point=10),
        budget=40, t_st=0, B=8, seed=2)
    save_serialized(
        "deep_lpp_epoch", deep, True, algo="lpp_sgd", Q=2, U=2, bounds=(0, int(e[2]), deep.dim),
        sched=rsched.LrSchedule(kind="cosine", alpha0=0.05, total=60, warmup=6, batch_local=8,
                                workers=2, batch_base=8, boost=True),
        sync=rsched.SyncScheme(total=60, period=4), budget=60, t_st=6, B=8, seed=1,
        epoch_partition=True)
    quad8 = robj.QuadraticObjective.from_dataset(rdata.make_linear_targets(32, 8, 1.0, 0.5, 3))
    save_serialized(
        "quad8_lpp", quad8, True, algo="lpp_sgd", Q=2, U=2, bounds=(0, 2, 4, 6, 8),
        sched=rsched.constant_schedule(0.05, 50), sync=rsched.SyncScheme(total=50, period=4),
        budget=50, t_st=8, B=8, seed=1)
    logreg8 = robj.LogisticObjective.from_dataset(rdata.make_blobs(64, 8, 2, 3.0, 0.5, 5))
    save_serialized(
        "logreg8_lap", logreg8, True, algo="lap_sgd", Q=2, U=2, bounds=(0, 8),
        sched=rsched.LrSchedule(kind="cosine", alpha0=0.1, total=60, warmup=6),
        sync=rsched.SyncScheme(total=60, period=4), budget=60, t_st=0, B=8, seed=2)
    c0_bounds = rpart.balanced_boundaries(c0.layer_param_counts, 2)
    save_serialized(
        "c0_lpp", c0, False, algo="lpp_sgd", Q=2, U=2, bounds=c0_bounds,
        sched=rsched.LrSchedule(kind="cosine", alpha0=0.05, total=200, warmup=20, batch_local=32,
                                workers=2, batch_base=32),
        sync=rsched.SyncScheme(total=200, period=16), budget=200, t_st=20, B=32, seed=1)

    # ---------------- BASELINE config 0: a small CNN in the reference's Objective protocol ----------------
    sys.path.insert(0, str(HERE.parents[1]))
    from oracle.cnn import SmallCnnOracle, make_images

    class RefCnn(robj.Objective):
        """The small CNN (oracle/cnn.py network math) plugged into the
        reference's Objective ABC, so the reference's own schedule primitives
        and engine drive it."""

        def __init__(self, o):
            self.o, self.dim, self.n_samples = o, o.dim, o.n_samples
            self.layer_param_counts = o.layer_param_counts

        def loss(self, x, batch):
            return self.o.loss(x, batch)

        def init_params(self, seed):
            return self.o.init_params(seed)

        def grad_block(self, x, block, batch):
            self.check_block(block)
            v = self.o.grad_block(x, block.start, block.stop, batch)
            return robj.GradResult(v, 0, 0, len(batch))

    cnn = RefCnn(SmallCnnOracle(*make_images(256, 3)))
    save_serialized(
        "cnn_lpp", cnn, True, algo="lpp_sgd", Q=2, U=2,
        bounds=rpart.balanced_boundaries(cnn.layer_param_counts, 2),
        sched=rsched.LrSchedule(kind="cosine", alpha0=0.05, total=40, warmup=4, batch_local=16,
                                workers=2, batch_base=16),
        sync=rsched.SyncScheme(total=40, period=4), budget=40, t_st=4, B=16, seed=1)
    cfg = rengine.RunConfig(
        algo="lap_sgd", objective=cnn, partition=rpart.make_partition(cnn.dim, (0, cnn.dim)),
        lr=rsched.constant_schedule(0.05, 30), sync=rsched.SyncScheme(total=30, period=4, switch_point=0),
        budget=30, warm_start_budget=0, workers=1, updaters=1, batch_size=16, seed=2,
        record_mode="full", quiescent=True)
    res = rengine.run_experiment(cfg)
    np.savez_compressed(HERE / "engine_cnn_q1u1.npz", final=res.final_values, x0=res.x0,
                        counter_finals=np.array(res.counter_finals))

    # ---------------- async band: the reference's own async runs of config C0 ----------------
    # (live threads: not deterministic, so the fixture is a band over seeds)
    band = {"config": "C0 MLP 3072-64-10, lpp_sgd Q=2 U=2 B=32 T=200, cosine 0.05 warmup 20, "
                      "T_st 20, period 16 after T/2, record light", "seeds": [], "initial": [], "final": []}
    for seed in (1, 2, 3, 4, 5):
        cfg = rengine.RunConfig(
            algo="lpp_sgd", objective=c0, partition=rpart.make_partition(c0.dim, c0_bounds),
            lr=rsched.LrSchedule(kind="cosine", alpha0=0.05, total=200, warmup=20, batch_local=32,
                                 workers=2, batch_base=32),
            sync=rsched.SyncScheme(total=200, period=16), budget=200, warm_start_budget=20,
            workers=2, updaters=2, batch_size=32, seed=seed, record_mode="light")
        res = rengine.run_experiment(cfg)
        band["seeds"].append(seed)
        band["initial"].append(res.metrics[0].train_loss)
        band["final"].append(res.metrics[-1].train_loss)
    (HERE / "async_band_c0.json").write_text(json.dumps(band, indent=1))

    # ---------------- the reference engine itself: Q=1, U=1, quiescent, full ----------------
    sched = rsched.constant_schedule(0.05, 50)
    cfg = rengine.RunConfig(
        algo="lap_sgd", objective=small, partition=rpart.make_partition(small.dim, (0, small.dim)),
        lr=sched, sync=rsched.SyncScheme(total=50, period=4, switch_point=0), budget=50,
        warm_start_budget=0, workers=1, updaters=1, batch_size=8, seed=1, record_mode="full",
        quiescent=True)
    res = rengine.run_experiment(cfg)
    np.savez_compressed(HERE / "engine_q1u1.npz", final=res.final_values, x0=res.x0,
                        counter_finals=np.array(res.counter_finals))
    # ---------------- event log + replay (instrumentation.py:166-219, 371-463) ----------------
    from asyncsgd import instrumentation as rinst

    cfg = rengine.RunConfig(
        algo="lpp_sgd", objective=deep, partition=rpart.make_partition(deep.dim, (0, int(e[2]), deep.dim)),
        lr=rsched.constant_schedule(0.05, 40), sync=rsched.SyncScheme(total=40, period=4, switch_point=8),
        budget=40, warm_start_budget=6, workers=2, updaters=2, batch_size=8, seed=3,
        record_mode="full", quiescent=True)
    res = rengine.run_experiment(cfg)
    import gzip

    tmp = Path("/tmp/eventlog_ref.ndjson")
    rinst.save_event_log(tmp, res)
    with open(tmp, "rb") as src, gzip.GzipFile(HERE / "eventlog_ref.ndjson.gz", "wb", mtime=0) as dst:
        dst.write(src.read())
    rep = rinst.replay_rounds(res)
    measured = [st.mean for st in sorted(res.stamps, key=lambda st: st.round) if st.worker == 0]
    np.savez_compressed(HERE / "eventlog_ref_replay.npz", round_means=np.stack(rep.round_means),
                        measured=np.stack(measured), x0=res.x0, distances=rep.distances,
                        clean=rep.clean, k_bar=np.array([rep.k_bar]))
    print("golden vectors written to", HERE)


if __name__ == "__main__":
    main()
