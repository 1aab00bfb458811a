"""Native (C++) vs Python updater + averager loops: minibatches/s,
images/s and averaging rounds/s on a host-bound tiny MLP, the config-0
small CNN and ResNet-20 (U=4, device sampling, record_mode off; CUDA-event
device time; sync period 1 for the first half, 16 after)."""
import dataclasses, json, sys
from pathlib import Path
import numpy as np
import torch
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench
from paper_2203_06638_b200.engine import Trainer
from paper_2203_06638_b200.objectives import MlpObjective, ResNetObjective

torch.backends.cudnn.benchmark = True
X = np.random.default_rng(0).normal(size=(4096, 16)).astype(np.float32)
cases = [("tiny_mlp", MlpObjective(X, np.arange(4096) % 4, (16, 16, 16), 4), 8, 4000),
         ("smallcnn", ResNetObjective("smallcnn", n_samples=8192, seed=0), 32, 2000),
         ("resnet20", ResNetObjective("resnet20", n_samples=50_000, seed=0), 128, 200)]
for name, obj, B, K in cases:
    for loop in ("python", "native"):
        cfg = dataclasses.replace(bench.build_cfg(obj, (K + 50) * 4), batch_size=B, host_loop=loop)
        tr = Trainer(cfg)
        tr.run(50 * 4, evaluate=False)
        torch.cuda.synchronize()
        r = tr.run(K * 4, evaluate=False)
        steps = sum(r.counter_finals)
        rounds = max((st.round for st in r.stamps), default=0)
        print(json.dumps({"model": name, "loop": loop, "native": tr.eng.native_loop(),
                          "native_averager": tr.eng.native_averager(), "B": B,
                          "rounds": rounds, "rounds_per_s": round(rounds / (r.device_ms / 1e3)),
                          "minibatches_per_s": round(steps / (r.device_ms / 1e3)),
                          "images_per_s": round(steps * B / (r.device_ms / 1e3))}), flush=True)
        tr.close()
