"""API records of a run — the reference's engine types (engine.py:34-150).

``RunConfig`` keeps the reference's fields, defaults and validation messages
(engine.py:34-72) and adds B200 options whose defaults preserve the
reference's semantics; ``UpdateRecord``, ``AveragerStamp``, ``MetricsRow``
and ``RunResult`` have the reference's fields (device tensors where the
reference has numpy arrays) plus timing extras on ``RunResult``.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import _native as N
from .objectives import ArenaObjective
from .partition import BlockPartition
from .schedules import LrSchedule, SyncScheme

ALGOS = ("mb_sgd", "pl_sgd", "lap_sgd", "lpp_sgd")


@dataclass(frozen=True)
class RunConfig:
    algo: str
    objective: ArenaObjective
    partition: BlockPartition
    lr: LrSchedule
    sync: SyncScheme
    budget: int
    warm_start_budget: int
    workers: int = 2
    updaters: int = 4
    batch_size: int = 32
    seed: int = 0
    eval_interval: int = 0
    record_mode: str = "light"
    tag_sample: int = 16
    quiescent: bool = False
    epoch_partition: bool = False
    round_budget: int | None = None
    # --- B200 extensions (defaults keep the reference's semantics) ---
    schedule: str = "async"          # "async" | "serialized" (canonical parity schedule)
    momentum: float = 0.0            # per-stream momentum buffers (paper: 0.9)
    weight_decay: float = 0.0
    apply_mode: str = "red"          # "red" | "bulk" | "plain" (plain may lose updates)
    sampling: str = "host"           # "host": reference rng stream, H2D per step; "device": in-graph
    devices: tuple[int, ...] | None = None   # in-process worker -> device map
    use_graphs: bool = True
    in_flight: int = 2
    evaluate: bool = True            # compute the initial/final MetricsRow losses
    averaging: str = "p2p"           # "p2p": owner-computes over peer arenas; "nvls": in-switch
    apply_priority: bool | None = None  # K1/K2 (or fused K1+K3) on a high-priority stream per
                                     # updater, ordered by events, so the apply is not queued behind
                                     # other streams' kernels; None = on for the native loop with
                                     # U <= 4 (in-situ apply -33 %, images/s neutral), off for the
                                     # Python loop (4 extra calls per step cost host time) and for
                                     # U > 4 (2U streams exceed the 8 hardware queues)
    fuse_snapshot: bool = True       # async: fuse each apply with the next step's snapshot
    track_writes: bool | None = None  # K5 write tags; None = reference default (lap/lpp)
    record_tensors: bool = True      # record_mode="full": keep per-update grad/snapshot copies
    host_loop: str = "auto"          # updater loop: "native" (C++, GIL-free), "python", "auto"

    @property
    def tracks(self) -> bool:
        if self.track_writes is not None:
            return bool(self.track_writes)
        return self.algo in ("lap_sgd", "lpp_sgd")

    def __post_init__(self):
        if self.algo not in ALGOS:
            raise ValueError(f"unknown algorithm {self.algo!r}")
        if self.algo in ("mb_sgd", "pl_sgd") and self.updaters != 1:
            raise ValueError(f"{self.algo} is sequential per worker; set updaters=1")
        if self.record_mode not in ("off", "light", "full"):
            raise ValueError(f"unknown record mode {self.record_mode!r}")
        if self.workers < 1 or self.updaters < 1 or self.batch_size < 1:
            raise ValueError("workers, updaters, batch_size must be positive")
        if self.budget < 1:
            raise ValueError("budget must be positive")
        if self.algo == "lpp_sgd" and self.partition.num_blocks < self.updaters:
            raise ValueError("need at least one block per updater")
        if self.round_budget is not None:
            if self.algo in ("mb_sgd", "pl_sgd"):
                raise ValueError("round_budget applies to asynchronous runs only")
            if self.round_budget < 1:
                raise ValueError("round_budget must be positive")
        if self.schedule not in ("async", "serialized"):
            raise ValueError(f"unknown schedule {self.schedule!r}")
        if self.apply_mode not in N.MODES:
            raise ValueError(f"unknown apply mode {self.apply_mode!r}")
        if self.sampling not in ("host", "device"):
            raise ValueError(f"unknown sampling {self.sampling!r}")
        if self.averaging not in ("p2p", "nvls"):
            raise ValueError(f"unknown averaging {self.averaging!r}")
        if self.host_loop not in ("auto", "native", "python"):
            raise ValueError(f"unknown host loop {self.host_loop!r}")
        if self.workers > N.MAX_WORKERS:
            raise ValueError(f"at most {N.MAX_WORKERS} workers per averaging group")


@dataclass(slots=True)
class UpdateRecord:
    worker: int
    rank: int
    s: int
    u: int
    k_claim: int
    block_id: int
    reason: str
    lr: float
    flops: int
    backward_flops: int
    clean: bool | None
    tag_indices: np.ndarray | None = None
    tags: np.ndarray | None = None
    grad: np.ndarray | None = None
    snapshot: np.ndarray | None = None


@dataclass(slots=True)
class AveragerStamp:
    worker: int
    round: int
    u: int
    s_cur: int
    k_delta: int
    wall_ms: float
    snapshot: np.ndarray | None = None
    mean: np.ndarray | None = None


@dataclass(frozen=True)
class MetricsRow:
    algo: str
    seed: int
    wall_ms: float
    samples: int
    round: int
    train_loss: float
    grad_norm_sq: float
    flops: int
    p_hat: float

    CSV_HEADER = "algo,seed,wall_ms,samples,round,train_loss,grad_norm_sq,flops,p_hat"

    def as_csv(self) -> str:
        return ",".join([self.algo, str(self.seed), repr(self.wall_ms), str(self.samples),
                         str(self.round), repr(self.train_loss), repr(self.grad_norm_sq),
                         str(self.flops), repr(self.p_hat)])


@dataclass
class RunResult:
    config: RunConfig
    metrics: list[MetricsRow]
    final_values: np.ndarray
    x0: np.ndarray
    wall_ms: float
    flops: int
    p_hat: float
    counter_finals: list[int]
    updates: list[UpdateRecord] = field(default_factory=list)
    stamps: list[AveragerStamp] = field(default_factory=list)
    device_ms: float = 0.0           # CUDA-event time of the run (first launch -> drain)
    apply_timing: tuple = ()          # (launches, total apply ms, algorithmic bytes) if timed


# ---------------------------------------------------------------------------
# round control block (host int64 cells; shared memory for multi-process)
