"""e2e (host batches + H2D + loss D2H) images/s vs in_flight depth."""
import dataclasses, json, sys
from pathlib import Path
import torch
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench
from paper_2203_06638_b200.engine import Trainer
from paper_2203_06638_b200.objectives import ResNetObjective

torch.backends.cudnn.benchmark = True
K = 60
obj = ResNetObjective("resnet20", n_samples=50_000, seed=0, data="host")
for inf in (2, 3, 4, 6):
    cfg = dataclasses.replace(bench.build_cfg(obj, (K + 5) * 4, sampling="host"), in_flight=inf)
    tr = Trainer(cfg, host_batches=True, read_loss=True)
    tr.run(20, evaluate=False)
    vals = []
    for _ in range(3):
        r = tr.run(K * 4, evaluate=False)
        vals.append(round(sum(r.counter_finals) * 128 / (r.device_ms / 1e3)))
    tr.close()
    print(json.dumps({"in_flight": inf, "e2e_img_s": vals}), flush=True)
