"""Engine-level knobs on the ResNet-20 LPP workload + host step-rate ceiling."""
import dataclasses, json, sys, time
from pathlib import Path
import torch
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench
from paper_2203_06638_b200.engine import Trainer
from paper_2203_06638_b200.objectives import MlpObjective, ResNetObjective

torch.backends.cudnn.benchmark = True
K, W = 40, 5


def measure(obj, B, **over):
    U = over.pop("updaters", 4)
    cfg = bench.build_cfg(obj, (K + W) * U, updaters=U)
    cfg = dataclasses.replace(cfg, batch_size=B, **over)
    tr = Trainer(cfg)
    tr.run(W * U, evaluate=False)
    torch.cuda.synchronize()
    res = tr.run(K * U, evaluate=False)
    tr.close()
    n = sum(res.counter_finals)
    return n / (res.device_ms / 1e3), n * B / (res.device_ms / 1e3)


obj = ResNetObjective("resnet20", n_samples=50_000, seed=0)
for kw in [dict(in_flight=2), dict(in_flight=3), dict(in_flight=4), dict(track_writes=False),
           dict(updaters=6), dict(apply_mode="bulk", track_writes=False)]:
    steps, imgs = measure(obj, 128, **dict(kw))
    print(json.dumps({"workload": "resnet20", **{k: str(v) for k, v in kw.items()},
                      "minibatch_per_s": round(steps), "img_per_s": round(imgs)}), flush=True)
import numpy as np
X = np.random.default_rng(0).normal(size=(256, 16)).astype(np.float32)
y = np.arange(256) % 4
tiny = MlpObjective(X, y, (16, 16, 16), 4)
for kw in [dict(in_flight=2), dict(in_flight=4), dict(track_writes=False, in_flight=4)]:
    steps, _ = measure(tiny, 8, **dict(kw))
    print(json.dumps({"workload": "tiny_mlp_host_ceiling", **{k: str(v) for k, v in kw.items()},
                      "minibatch_per_s": round(steps)}), flush=True)
