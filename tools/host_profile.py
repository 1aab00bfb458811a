"""Host-side cost per updater step (tiny model => host-bound): minibatches/s
and a cProfile of one updater thread."""
import cProfile, dataclasses, io, pstats, sys, threading
from pathlib import Path
import numpy as np
import torch
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench
from paper_2203_06638_b200 import engine as E
from paper_2203_06638_b200.objectives import MlpObjective

X = np.random.default_rng(0).normal(size=(256, 16)).astype(np.float32)
tiny = MlpObjective(X, np.arange(256) % 4, (16, 16, 16), 4)
cfg = dataclasses.replace(bench.build_cfg(tiny, 2000 * 4), batch_size=8, sampling="host")
tr = E.Trainer(cfg)
tr.run(200, evaluate=False)
r = tr.run(2000 * 4, evaluate=False)
print("minibatches/s", round(sum(r.counter_finals) / (r.wall_ms / 1e3)))
prof = cProfile.Profile()
orig = tr.eng.updater


def profiled(q, rr):
    if rr == 0:
        prof.enable()
        try:
            orig(q, rr)
        finally:
            prof.disable()
    else:
        orig(q, rr)


tr.eng.updater = profiled
tr.run(1000 * 4, evaluate=False)
s = io.StringIO()
pstats.Stats(prof, stream=s).sort_stats("tottime").print_stats(18)
print(s.getvalue()[:4000])
