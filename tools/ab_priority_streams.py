"""Apply-stream priority vs the number of hardware work queues: ResNet-20
LPP-SGD images/s at U = 4 / 6 with apply_priority off/on (each updater adds
a second stream when on).  Run once with the default 8 connections and once
with CUDA_DEVICE_MAX_CONNECTIONS=32."""
import dataclasses, json, os, sys
from pathlib import Path
import torch
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench
from paper_2203_06638_b200.engine import Trainer
from paper_2203_06638_b200.objectives import ResNetObjective

torch.backends.cudnn.benchmark = True
obj = ResNetObjective("resnet20", n_samples=50_000, seed=0)
conn = os.environ.get("CUDA_DEVICE_MAX_CONNECTIONS", "8 (default)")
for U in (4, 6):
    res = {False: [], True: []}
    for rep in range(3):
        for p in (False, True):
            K = 100
            cfg = dataclasses.replace(bench.build_cfg(obj, (K + 5) * U, updaters=U), apply_priority=p)
            tr = Trainer(cfg)
            tr.run(5 * U, evaluate=False)
            r = tr.run(K * U, evaluate=False)
            res[p].append(round(sum(r.counter_finals) * 128 / (r.device_ms / 1e3)))
            tr.close()
    print(json.dumps({"connections": conn, "U": U, "priority_off": res[False], "priority_on": res[True]}),
          flush=True)
