"""Locate the e2e gap: device data + host indices; host batches without loss D2H; full e2e."""
import dataclasses, json, sys
from pathlib import Path
import torch
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench
from paper_2203_06638_b200.engine import Trainer
from paper_2203_06638_b200.objectives import ResNetObjective

torch.backends.cudnn.benchmark = True
K = 60
dev_obj = ResNetObjective("resnet20", n_samples=50_000, seed=0, data="device")
host_obj = ResNetObjective("resnet20", n_samples=50_000, seed=0, data="host")
cases = [("device data, in-graph rng", dev_obj, "device", False, False),
         ("device data, host rng indices (H2D idx)", dev_obj, "host", False, False),
         ("host batches, no loss D2H", host_obj, "host", True, False),
         ("host batches + loss D2H (e2e)", host_obj, "host", True, True)]
for name, obj, sampling, hb, rl in cases:
    cfg = bench.build_cfg(obj, (K + 5) * 4, sampling=sampling)
    tr = Trainer(cfg, host_batches=hb, read_loss=rl)
    tr.run(20, evaluate=False)
    vals = []
    for _ in range(3):
        r = tr.run(K * 4, evaluate=False)
        vals.append(round(sum(r.counter_finals) * 128 / (r.device_ms / 1e3)))
    tr.close()
    print(json.dumps({"case": name, "img_s": vals}), flush=True)
