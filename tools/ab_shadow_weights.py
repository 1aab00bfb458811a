"""bf16 shadow weights (one cast kernel per step, model in native bf16) vs
autocast (per-tensor casts of every conv / linear weight in forward and of
every weight gradient in backward): ResNet-20 LPP U=4 images/s, and the
gradients of one step compared between the two."""
import dataclasses, json, sys
from pathlib import Path
import numpy as np
import torch
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench
from paper_2203_06638_b200.engine import Trainer
from paper_2203_06638_b200.objectives import ResNetObjective
from paper_2203_06638_b200.partition import Block

torch.backends.cudnn.benchmark = True
res = {True: [], False: []}
for rep in range(3):
    for sw in (False, True):
        obj = ResNetObjective("resnet20", n_samples=50_000, seed=0, shadow_weights=sw)
        K = 100
        tr = Trainer(bench.build_cfg(obj, (K + 5) * 4))
        tr.run(20, evaluate=False)
        r = tr.run(K * 4, evaluate=False)
        res[sw].append(round(sum(r.counter_finals) * 128 / (r.device_ms / 1e3)))
        tr.close()
# same step, both ways
torch.backends.cudnn.deterministic = True
x = ResNetObjective("resnet20", n_samples=512, seed=0).init_params(0)
g = {}
for sw in (False, True):
    o = ResNetObjective("resnet20", n_samples=512, seed=0, shadow_weights=sw)
    g[sw] = o.grad_block(x, Block(0, o.dim), np.arange(128)).values.cpu().numpy()
d = np.abs(g[True] - g[False])
print(json.dumps({"autocast": res[False], "shadow": res[True], "grad_max_abs_diff": float(d.max()),
                  "grad_bitwise_equal": bool((d == 0).all()), "grad_max_abs": float(np.abs(g[False]).max())}))
