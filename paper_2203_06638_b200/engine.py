"""LPP-SGD / LAP-SGD engine on B200, plus the MB-SGD / PL-SGD baselines.

Drop-in for ``asyncsgd.engine`` (``/root/reference/pkg/src/asyncsgd/engine.py``):
the same ``RunConfig`` (engine.py:34-72, same validation messages),
``run_experiment(cfg) -> RunResult`` (engine.py:637-642), ``UpdateRecord``,
``AveragerStamp``, ``MetricsRow``.  The execution model is B200-native:

* worker q = one GPU (or, in-process, one arena on a device) holding the
  shared fp32 arena x_q (``ParamStore``);
* updater r of worker q = one CUDA stream driven by one host thread; each
  step claims slot s from the host atomic counter C^q (engine.py:336),
  picks lr and the PASSM+ block (engine.py:337-342), then enqueues
  K3 snapshot -> captured fwd/bwd graph of that block -> K1/K2 apply on its
  stream (engine.py:343-355).  Updaters never block on the averager;
  in-flight steps per stream are bounded (``in_flight``) so the slot
  counter tracks device progress;
* averager of worker q = one host thread + a high-priority stream.  Round
  opening follows engine.py:394-412 (any worker's trigger opens the round
  for all, CAS-elected), and each round is one K4 launch over the shard
  this worker OWNS, which reads the shard from all Q arenas (peer / NVLink)
  and adds ``mean - v_q`` into every arena in place (engine.py:418-421)
  while updaters keep writing.  Averagers (never updaters) exchange one
  final-flag vote per round so that they stop on the same unanimous round
  (engine.py:452-453).

``schedule="serialized"`` runs the canonical deterministic interleaving
(oracle/schedule.py) with the very same step and round kernels;
it is the parity mode.

Modules: ``records`` (the API types), ``async_engine`` (workers, updater /
averager threads, serialized mode), ``sync_engine`` (MB / PL baselines);
this module keeps ``Trainer`` / ``run_experiment`` and re-exports the rest.

Multi-process groups (one process per GPU) attach through
``paper_2203_06638_b200.group`` (IPC arena mapping + a shared-memory
control block); in one process, Q workers may share one device (used by the
parity tests) or spread over the visible devices.
"""

from __future__ import annotations

import torch

from .async_engine import PauseGate, _Engine, shard_bounds  # noqa: F401
from .partition import Block
from .records import (ALGOS, AveragerStamp, MetricsRow, RunConfig, RunResult,  # noqa: F401
                      UpdateRecord)
from .rounds import RoundControl  # noqa: F401
from .sync_engine import _SyncEngine

__all__ = ["ALGOS", "RunConfig", "RunResult", "UpdateRecord", "AveragerStamp", "MetricsRow",
           "Trainer", "run_experiment", "shard_bounds", "PauseGate"]


# ---------------------------------------------------------------------------
# public entry point


def _eval_row(cfg, samples, rnd, wall_ms, flops, p_hat, x, evaluate: bool = True) -> MetricsRow:
    """engine.py:526-541: losses are computed post hoc, outside wall time."""
    obj = cfg.objective
    if evaluate:
        g = obj.full_grad(x)
        loss = obj.full_loss(x)
        gn = float((g.double() ** 2).sum())
    else:
        loss, gn = float("nan"), float("nan")
    return MetricsRow(algo=cfg.algo, seed=cfg.seed, wall_ms=wall_ms, samples=samples, round=rnd,
                      train_loss=loss, grad_norm_sq=gn, flops=flops, p_hat=p_hat)


class Trainer:
    """Public session API: build once (arenas, captured graphs), run phases.

    ``Trainer(cfg).run()`` is ``run_experiment(cfg)``; ``run(budget)`` may be
    called repeatedly (bench warm-up, then timed phase) on the same arenas.
    ``host_batches`` feeds every step from host (pinned) memory with an H2D
    copy inside the step; ``read_loss`` copies each step's loss back.
    """

    def __init__(self, cfg: RunConfig, group=None, host_batches: bool = False,
                 time_apply: bool = False, read_loss: bool = False):
        if not torch.cuda.is_available():
            raise RuntimeError("paper_2203_06638_b200 needs a CUDA device (no CPU fallback)")
        self.cfg = cfg
        self.sync = cfg.algo in ("mb_sgd", "pl_sgd")
        if self.sync:
            self.eng = _SyncEngine(cfg, group=group, host_batches=host_batches)
        else:
            self.eng = _Engine(cfg, host_batches=host_batches, time_apply=time_apply, group=group)
            self.eng.read_loss = read_loss
        self.phases = 0

    def run(self, budget: int | None = None, evaluate: bool | None = None) -> RunResult:
        cfg = self.cfg
        budget = cfg.budget if budget is None else int(budget)
        ev = cfg.evaluate if evaluate is None else evaluate
        eng = self.eng
        if self.sync:
            dev_ms = eng.run(budget)
            final = eng.final_values()
            fwd = cfg.objective.forward_cost()
            flops = budget * cfg.workers * cfg.batch_size * (
                fwd + cfg.objective.backward_cost(Block(0, cfg.objective.dim)))
            rounds = budget if cfg.algo == "mb_sgd" else eng.rounds
            rows = [_eval_row(cfg, 0, 0, 0.0, 0, 1.0, eng.x0_host, ev)]
            per_step = flops // budget
            rows += [_eval_row(cfg, k, j, wl, per_step * k, 1.0, xv.cpu().numpy(), ev)
                     for k, j, wl, _f, xv in eng.evals if k != budget]
            rows.append(_eval_row(cfg, budget, rounds, eng.wall_ms, flops, 1.0, final, ev))
            self.phases += 1
            return RunResult(config=cfg, metrics=rows, final_values=final, x0=eng.x0_host,
                             wall_ms=eng.wall_ms, flops=flops, p_hat=1.0,
                             counter_finals=[budget] * cfg.workers, device_ms=dev_ms)
        if self.phases:
            eng.reset(budget)
        else:
            eng.budget = budget
        self.phases += 1
        dev_ms = eng.run_serialized() if cfg.schedule == "serialized" else eng.run_async()
        final = eng.final_values()
        stamps = [st for per in eng.stamps for st in per]
        rounds = max((st.round for st in stamps), default=0)
        flops = eng.flops.read()
        counters = [eng.workers[q].store.sample_counter.read() for q in eng.local_workers]
        rows = [_eval_row(cfg, 0, 0, 0.0, 0, 1.0, eng.x0_host, ev)]
        rows += [_eval_row(cfg, sc, j, wl, fl, ph, m.cpu().numpy(), ev)
                 for sc, j, wl, fl, ph, m in eng.eval_points]
        rows.append(_eval_row(cfg, max(counters), rounds, eng.wall_ms, flops, eng.p_hat(), final, ev))
        res = RunResult(config=cfg, metrics=rows, final_values=final, x0=eng.x0_host,
                        wall_ms=eng.wall_ms, flops=flops, p_hat=eng.p_hat(), counter_finals=counters,
                        updates=[u for per in eng.updates for u in per], stamps=stamps,
                        device_ms=dev_ms, apply_timing=eng.apply_timing())
        res.round_trace = getattr(eng, "round_trace", None)
        res.losses = list(eng.loss_log)
        res.k4_timing = tuple(getattr(eng, "k4_timing", (0, 0.0)))   # (rounds, summed ms), in situ
        res.apply_ms_samples = list(getattr(eng, "apply_ms_samples", []))
        return res

    def close(self) -> None:
        self.eng.close()


def run_experiment(cfg: RunConfig, group=None, host_batches: bool = False) -> RunResult:
    """Run one configuration (engine.py:637-642).  ``group`` attaches this
    process to a multi-GPU group (``paper_2203_06638_b200.group``)."""
    tr = Trainer(cfg, group=group, host_batches=host_batches)
    try:
        return tr.run()
    finally:
        tr.close()
