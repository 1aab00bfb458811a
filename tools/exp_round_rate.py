"""Averaging-round rate of the native round protocol with Q in-process
workers on one GPU (tiny MLP, U = 1, averaging every tick): rounds/s with
write tags (fence 1 + the device round cell per round) and without (no
fence), Q = 2 / 4 / 8 — the host-protocol cost the N > 1 runs pay."""
import json
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from oracle import data as odata  # noqa: E402
from paper_2203_06638_b200.engine import RunConfig, run_experiment  # noqa: E402
from paper_2203_06638_b200.objectives import MlpObjective  # noqa: E402
from paper_2203_06638_b200.partition import make_partition  # noqa: E402
from paper_2203_06638_b200.schedules import SyncScheme, constant_schedule  # noqa: E402

X, y = odata.make_blobs(256, 16, 4, 2.0, 0.5, 3)
obj = MlpObjective(X, y, (16, 16), 4)
for Q in (2, 4, 8):
    for tags in (False, True):
        T = 1500
        cfg = RunConfig(algo="lap_sgd", objective=obj, partition=make_partition(obj.dim, (0, obj.dim)),
                        lr=constant_schedule(0.01, T), sync=SyncScheme(total=T, period=1, switch_point=T),
                        budget=T, warm_start_budget=0, workers=Q, updaters=1, batch_size=8, seed=1,
                        evaluate=False, record_mode="off", track_writes=tags, sampling="device")
        t0 = time.perf_counter()
        res = run_experiment(cfg)
        wall = time.perf_counter() - t0
        rounds = max(st.round for st in res.stamps)
        print(json.dumps({"Q": Q, "tags": tags, "rounds": rounds, "run_wall_ms": round(res.wall_ms, 1),
                          "rounds_per_s": round(rounds / (res.wall_ms / 1e3)),
                          "minibatches_per_s": round(sum(res.counter_finals) / (res.wall_ms / 1e3))}),
              flush=True)
