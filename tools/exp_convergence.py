"""Which factor separates async LPP from MB-SGD on a learnable CNN task?"""
import dataclasses, sys
from pathlib import Path
import torch
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "tests"))
from test_engine_gpu import _tiny
from paper_2203_06638_b200.engine import run_experiment
from paper_2203_06638_b200.objectives import ResNetObjective
from paper_2203_06638_b200.partition import balanced_boundaries, make_partition
from paper_2203_06638_b200.schedules import LrSchedule, SyncScheme

torch.backends.cudnn.benchmark = True
obj = ResNetObjective("resnet20", n_samples=2048, seed=0, pattern_scale=0.5)
slots = 160
full = make_partition(obj.dim, (0, obj.dim))
four = make_partition(obj.dim, balanced_boundaries(obj.layer_param_counts, 4))
base = _tiny(obj, algo="lpp_sgd", budget=slots, workers=1, updaters=4, batch_size=64, partition=four,
             warm_start_budget=16, momentum=0.9, weight_decay=5e-4, sampling="device",
             lr=LrSchedule(kind="cosine", alpha0=0.05, total=slots + 4, warmup=16),
             sync=SyncScheme(total=slots, period=16), evaluate=True)
cases = {
    "mb_sgd": dict(algo="mb_sgd", updaters=1, budget=slots + 4, partition=full, warm_start_budget=0),
    "lap_u1": dict(algo="lap_sgd", updaters=1, budget=slots + 3, partition=full),
    "lap_u4": dict(algo="lap_sgd", partition=full),
    "lpp_u4": dict(),
    "lpp_u4_nomom": dict(momentum=0.0),
    "lap_u4_nomom": dict(algo="lap_sgd", partition=full, momentum=0.0),
    "mb_nomom": dict(algo="mb_sgd", updaters=1, budget=slots + 4, partition=full, warm_start_budget=0, momentum=0.0),
}
for name, over in cases.items():
    r = run_experiment(dataclasses.replace(base, **over))
    print(f"{name:14s} loss {r.metrics[0].train_loss:.3f} -> {r.metrics[-1].train_loss:.3f}  minibatches {sum(r.counter_finals) if name[:2] != 'mb' else r.counter_finals[0]}", flush=True)
